mkdir -p gpurun_out/d20
SIDA_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/d20/ep2.json 2> gpurun_out/d20/ep2.err; echo ep2=$?
tail -c 1500 gpurun_out/d20/ep2.json; tail -5 gpurun_out/d20/ep2.err
SIDA_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --impl reference > gpurun_out/d20/ref2.json 2> gpurun_out/d20/ref2.err; echo ref2=$?
head -c 600 gpurun_out/d20/ref2.json
