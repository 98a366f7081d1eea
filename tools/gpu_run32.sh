mkdir -p gpurun_out
python -m pytest -q -m gpu tests > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
python bench.py --particles 256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b256.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b256_v2.csv python bench.py --particles 256 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/status.txt
