mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err; echo "bench=$?" > gpurun_out/s_status.txt
export BMB_NO_WARMUP=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"build_xi_pair" --launch-skip 5 --launch-count 1 -o gpurun_out/xi_pair2 python tools/probe_bands.py 64 > gpurun_out/ncu_xi.log 2>&1; echo ncu_xi=$? >> gpurun_out/s_status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"seed_kernel" --launch-skip 1 --launch-count 1 -o gpurun_out/seed2 python tools/probe_bands.py 64 > gpurun_out/ncu_seed.log 2>&1; echo ncu_seed=$? >> gpurun_out/s_status.txt
