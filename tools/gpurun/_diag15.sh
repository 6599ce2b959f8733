P="python tools/ffn_probe.py --iters 20 --no-cublas"
echo "== bal 128"; SIDA_GEMM_PROF=1 $P --experts 128
echo "== bal 128 PDL0"; SIDA_PDL=0 SIDA_GEMM_PROF=1 $P --experts 128
echo "== bal 8"; SIDA_GEMM_PROF=1 $P --experts 8
