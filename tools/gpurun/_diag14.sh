{
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "ffn" 2>&1 | tail -2
P="python tools/ffn_probe.py --iters 20 --no-cublas"
echo "== bal 128"; SIDA_GEMM_PROF=1 $P --experts 128
echo "== bal 128 CG1"; SIDA_FFN_CG=1 $P --experts 128
echo "== bal 128 TN"; SIDA_FFN_SWAP=1 $P --experts 128
echo "== bal 128 TN2"; SIDA_FFN_SWAP=2 $P --experts 128
echo "== exact 128"; $P --experts 128 --exact
echo "== bal 64"; $P --experts 64
echo "== bal 256"; $P --experts 256
echo "== bal 8"; $P --experts 8
echo "== 131k"; $P --experts 128 --tokens 131072 --iters 10
} 2>&1
