for r in 1 2; do
for E in 128 64 256 8; do
  for M in -1 1 2 3; do echo "E=$E swap=$M $(SIDA_FFN_SWAP=$M python tools/ffn_probe.py --experts $E --iters 20 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3)"; done
  echo "E=$E xffn $(SIDA_XFFN=1 python tools/ffn_probe.py --experts $E --iters 20 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3)"
done
done
echo "131k swap=-1 $(python tools/ffn_probe.py --experts 128 --tokens 131072 --iters 10 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3)"
echo "131k swap=1 $(SIDA_FFN_SWAP=1 python tools/ffn_probe.py --experts 128 --tokens 131072 --iters 10 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3)"
echo "131k xffn $(SIDA_XFFN=1 python tools/ffn_probe.py --experts 128 --tokens 131072 --iters 10 --no-cublas 2>&1 | grep 'ffn layer' | cut -d' ' -f3)"
