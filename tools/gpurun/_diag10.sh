mkdir -p gpurun_out/d10
P="python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas --exact"
{
echo "== exact auto(CG1)"; $P
echo "== exact CG2"; SIDA_FFN_CG=2 $P
echo "== exact TN"; SIDA_FFN_SWAP=1 $P
echo "== exact xffn"; SIDA_XFFN=1 SIDA_XFFN_PROF=1 $P
echo "== exact xffn diag1"; SIDA_XFFN=1 SIDA_XFFN_DIAG=1 SIDA_XFFN_PROF=1 $P
echo "== exact 64 CG2"; SIDA_FFN_CG=2 python tools/ffn_probe.py --experts 64 --iters 20 --no-cublas --exact
echo "== exact 64 xffn"; SIDA_XFFN=1 python tools/ffn_probe.py --experts 64 --iters 20 --no-cublas --exact
} > gpurun_out/d10/out.txt 2>&1
cat gpurun_out/d10/out.txt
