mkdir -p gpurun_out
python bench.py --particles 256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b256.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b256_v2.csv python bench.py --particles 256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$? > gpurun_out/status.txt
python tools/probe_align.py 64 > gpurun_out/probe64.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:expand_factored -s 1 -c 1 -o gpurun_out/r1b_expand python tools/probe_align.py 64 > gpurun_out/ncu_e.log 2>&1; echo ncu2=$? >> gpurun_out/status.txt
python tools/probe_refine_l16.py 64 > gpurun_out/refine_l16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"eval_kernel|compose_kernel" -c 3 -o gpurun_out/r1b_refine python tools/probe_refine_l16.py 64 > gpurun_out/ncu_r.log 2>&1; echo ncu3=$? >> gpurun_out/status.txt
