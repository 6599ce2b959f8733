P="python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas"
for D in 0 1 2 3; do echo "== exact diag $D"; SIDA_XFFN=1 SIDA_XFFN_DIAG=$D SIDA_XFFN_PROF=1 $P --exact; done
for D in 0 1 2 3; do echo "== bal diag $D"; SIDA_XFFN=1 SIDA_XFFN_DIAG=$D $P; done
