# ncu of one config-2 expansion launch of the quad-copy pair-list kernel:
#   gpurun --timeout 1500 -- 'bash tools/gpu_ncu_quad.sh'
mkdir -p gpurun_out
export BMB_NO_WARMUP=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"expand_quad" --launch-skip 1 --launch-count 1 -o gpurun_out/expand_quad python tools/probe_bands.py 64 > gpurun_out/ncu_quad.log 2>&1; echo ncu_quad=$? > gpurun_out/status_ncu_quad.txt
