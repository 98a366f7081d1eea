mkdir -p gpurun_out
set -x
python bench.py --particles 256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b256.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b256.csv python bench.py --particles 256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/status.txt
ncu --set full --clock-control none --import-source on -k regex:expand_factored -s 2 -c 1 -o gpurun_out/expand_full python bench.py --particles 256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$? >> gpurun_out/status.txt
ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 40 -c 2 -o gpurun_out/evalk_full python bench.py --particles 256 --steps 1 --warmup 3 --no-cpu-baseline >> gpurun_out/ncu_full.log 2>&1; echo ncu3=$? >> gpurun_out/status.txt
