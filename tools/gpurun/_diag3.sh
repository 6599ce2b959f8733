mkdir -p gpurun_out/d3
python tools/cublas_probe.py 128 > gpurun_out/d3/cublas.txt 2>&1
python tools/cublas_probe.py 8 >> gpurun_out/d3/cublas.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"nvjet|cutlass|gemm|sm100" -s 6 -c 4 -o gpurun_out/d3/cublas128 python tools/cublas_probe.py 128 > gpurun_out/d3/ncu.log 2>&1
cat gpurun_out/d3/cublas.txt
