# Quick GPU check: tests, smoke, a bench line and the reference arm.
mkdir -p gpurun_out/q
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/q/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/q/gputests.log 2>&1; echo tests=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/q/bench.json 2> gpurun_out/q/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/q/bench_ref.json 2> gpurun_out/q/bench_ref.err; echo ref=$?
tail -5 gpurun_out/q/gputests.log; tail -2 gpurun_out/q/smoke.log; cat gpurun_out/q/bench.json | head -c 3000
