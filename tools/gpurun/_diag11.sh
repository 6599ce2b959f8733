mkdir -p gpurun_out/d11
{
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "grouped_ffn_bf16_vs_oracle or one_launch" 2>&1 | tail -2
P="python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas"
echo "== exact xffn"; SIDA_XFFN=1 SIDA_XFFN_PROF=1 $P --exact
echo "== bal xffn"; SIDA_XFFN=1 SIDA_XFFN_PROF=1 $P
echo "== bal auto"; $P
echo "== exact 64 xffn"; SIDA_XFFN=1 python tools/ffn_probe.py --experts 64 --iters 20 --no-cublas --exact
echo "== bal 256 xffn"; SIDA_XFFN=1 python tools/ffn_probe.py --experts 256 --iters 20 --no-cublas
} > gpurun_out/d11/out.txt 2>&1
cat gpurun_out/d11/out.txt
