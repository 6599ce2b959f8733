mkdir -p gpurun_out/d7
{
echo "== split auto 128"; SIDA_GEMM_PROF=1 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas
echo "== CG1 128"; SIDA_FFN_CG=1 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas
echo "== split 128 again"; python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas
echo "== split 64"; python tools/ffn_probe.py --experts 64 --iters 20 --no-cublas
echo "== CG1/2 64"; SIDA_FFN_CG=2 python tools/ffn_probe.py --experts 64 --iters 20 --no-cublas
echo "== split 256"; python tools/ffn_probe.py --experts 256 --iters 20 --no-cublas
echo "== old 256"; SIDA_FFN_CG=1 python tools/ffn_probe.py --experts 256 --iters 20 --no-cublas
echo "== 131k"; python tools/ffn_probe.py --experts 128 --tokens 131072 --iters 10 --no-cublas
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none -k regex:"grouped_gemm" -s 6 -c 4 -o gpurun_out/d7/split128 python tools/ffn_probe.py --experts 128 --iters 3 --no-cublas > /dev/null 2>&1
} > gpurun_out/d7/out.txt 2>&1
cat gpurun_out/d7/out.txt
