# per-GEMM launch times of both tile families over the expert-count / batch grid
for KT in 8:32768 32:32768 64:32768 128:32768 256:32768 256:1024 256:4096 256:16384 128:131072; do
K=${KT%%:*}; T=${KT##*:}
for S in 0 1; do
SIDA_FFN_SWAP=$S timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"grouped_gemm" -s 8 -c 2 --csv python tools/ffn_probe.py --experts $K --tokens $T --iters 1 --no-cublas 2>/dev/null | grep gpu__time | awk -F'","' -v k=$K -v t=$T -v s=$S '{print "K=" k " T=" t " swap=" s " " substr($5,1,30) " " $NF}'
done; done
