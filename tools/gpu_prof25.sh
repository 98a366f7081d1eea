# CUPTI kernel profiles of one config-2 and one config-5 step (1024 / 512 particles, 4 lanes)
mkdir -p gpurun_out
timeout 600 python tools/profile_kernels.py 1024 4 > gpurun_out/prof_cfg2.txt 2>&1
CONFIG=5 timeout 600 python tools/profile_kernels.py 512 4 > gpurun_out/prof_cfg5.txt 2>&1
