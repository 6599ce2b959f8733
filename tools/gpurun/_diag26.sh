mkdir -p gpurun_out/sw
timeout 1500 python tools/sweep.py --experts 256 --batches 1,8,64,256,512 --seqs 128,256,512 --max-tokens 262144 --out gpurun_out/sw/sweep_base256.json > gpurun_out/sw/base256.log 2>&1; echo sw256=$?
timeout 900 python tools/sweep.py --experts 8 --batches 1,8,64,256 --seqs 128,512 --out gpurun_out/sw/sweep_base8.json > gpurun_out/sw/base8.log 2>&1; echo sw8=$?
tail -20 gpurun_out/sw/base256.log
