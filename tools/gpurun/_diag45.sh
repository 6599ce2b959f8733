for L in 25 12 48; do
echo "lag $L: bal $(SIDA_XFFN=1 SIDA_XFFN_LAG=$L python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3) exact $(SIDA_XFFN=1 SIDA_XFFN_LAG=$L python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas --exact 2>&1 | grep 'ffn layer' | cut -d' ' -f3)"
done
echo "TN bal $(python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3)"
echo "xffn 64 $(SIDA_XFFN=1 python tools/ffn_probe.py --experts 64 --iters 20 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3) TN 64 $(python tools/ffn_probe.py --experts 64 --iters 20 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3)"
echo "xffn 256 $(SIDA_XFFN=1 python tools/ffn_probe.py --experts 256 --iters 20 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3) TN 256 $(python tools/ffn_probe.py --experts 256 --iters 20 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3)"
