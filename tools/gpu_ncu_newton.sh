mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"step_kernel|accept_kernel" --launch-skip 40 --launch-count 4 -o gpurun_out/newton_l16 python tools/probe_bands.py 64 > gpurun_out/ncu_newton.log 2>&1; echo ncu=$? > gpurun_out/status.txt
