mkdir -p gpurun_out/d2
P="python tools/ffn_probe.py --experts 128 --iters 20"
{
echo "== auto"; SIDA_GEMM_PROF=1 $P
echo "== swap0 (token-M both)"; SIDA_FFN_SWAP=0 SIDA_GEMM_PROF=1 $P --no-cublas
echo "== swap1 (token-N both)"; SIDA_FFN_SWAP=1 SIDA_GEMM_PROF=1 $P --no-cublas
echo "== swap2"; SIDA_FFN_SWAP=2 SIDA_GEMM_PROF=1 $P --no-cublas
echo "== xffn"; SIDA_XFFN=1 SIDA_XFFN_PROF=1 $P --no-cublas
echo "== alias4 auto"; SIDA_GEMM_PROF=1 $P --no-cublas --alias-slots 4
echo "== alias4 xffn"; SIDA_XFFN=1 SIDA_XFFN_PROF=1 $P --no-cublas --alias-slots 4
echo "== base8 auto"; SIDA_GEMM_PROF=1 python tools/ffn_probe.py --experts 8 --iters 20
echo "== 131k auto"; SIDA_GEMM_PROF=1 python tools/ffn_probe.py --experts 128 --tokens 131072 --iters 10 --no-cublas
} > gpurun_out/d2/ffn.txt 2>&1
cat gpurun_out/d2/ffn.txt
