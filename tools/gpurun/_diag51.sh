mkdir -p gpurun_out/d51
SIDA_BENCH_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 3 --warmup 3 --no-extras > gpurun_out/d51/ep4.json 2> gpurun_out/d51/ep4.err; echo ep4=$?
python -c "import json; d=json.load(open('gpurun_out/d51/ep4.json')); print(d['config']['parallelism'], d['n_gpus'], round(d['value']/1e6,3), d['gpu_launches'])"
tail -3 gpurun_out/d51/ep4.err
