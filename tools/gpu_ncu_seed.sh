# ncu of one config-2 seed launch and one window/side kernel build
mkdir -p gpurun_out
export BMB_NO_WARMUP=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"seed_kernel" --launch-skip 1 --launch-count 1 -o gpurun_out/seed python tools/probe_bands.py 64 > gpurun_out/ncu_seed.log 2>&1; echo ncu_seed=$? > gpurun_out/status_ncu_seed.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"build_xi_pair" --launch-skip 5 --launch-count 1 -o gpurun_out/xi_pair python tools/probe_bands.py 64 > gpurun_out/ncu_xi.log 2>&1; echo ncu_xi=$? >> gpurun_out/status_ncu_seed.txt
