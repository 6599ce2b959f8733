mkdir -p gpurun_out/d12
{
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
P="python tools/ffn_probe.py --iters 20 --no-cublas"
for E in 128 64 256 8; do echo "== bal $E (CG2+half)"; SIDA_GEMM_PROF=1 $P --experts $E; echo "== bal $E CG1"; SIDA_FFN_CG=1 $P --experts $E; done
echo "== exact 128"; $P --experts 128 --exact
echo "== 131k"; $P --experts 128 --tokens 131072 --iters 10
timeout 600 ncu --set full --clock-control none -k regex:"grouped_gemm" -s 4 -c 2 -o gpurun_out/d12/half128 python tools/ffn_probe.py --experts 128 --iters 3 --no-cublas > /dev/null 2>&1
} > gpurun_out/d12/out.txt 2>&1
cat gpurun_out/d12/out.txt
