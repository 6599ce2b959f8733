# token-M STAGE-2 epilogue, second pass (lookahead only for BN <= 192): full GPU suite + probes
mkdir -p gpurun_out/epi2
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/epi2/tests.txt 2>&1; echo tests=$?
tail -2 gpurun_out/epi2/tests.txt
for r in 1 2; do
for v in old new; do
  cp ab_$v.so paper_2310_18859_b200/_sida_b200.so
  echo "== $v run $r"
  timeout 120 python tools/proj_probe.py
  SIDA_FFN_SWAP=0 timeout 120 python tools/ffn_probe.py --experts 8 --no-cublas
  timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas
done
done 2>&1 | tee gpurun_out/epi2/ab.txt
cp ab_new.so paper_2310_18859_b200/_sida_b200.so
