mkdir -p gpurun_out
set -x
python -m pytest -q -m gpu tests > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$? >> gpurun_out/status.txt
python bench.py --particles 64 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --particles 64 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/status.txt
ncu --set full --clock-control none --import-source on -k regex:split3 -s 2 -c 1 -o gpurun_out/gemm_full python bench.py --particles 64 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$? >> gpurun_out/status.txt
