{
P="python tools/ffn_probe.py --iters 20 --no-cublas"
echo "== bal 128"; SIDA_GEMM_PROF=1 $P --experts 128
echo "== exact 128"; SIDA_GEMM_PROF=1 $P --experts 128 --exact
echo "== bal 8"; SIDA_GEMM_PROF=1 $P --experts 8
} 2>&1
