# Round-2 GPU evidence pass: tests, smoke, bench (both arms), launch list, ncu of the hot kernels.
bash tools/_gpu_quick.sh
bash tools/_profile_r2.sh
