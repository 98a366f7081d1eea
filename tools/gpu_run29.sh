mkdir -p gpurun_out
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
python tools/probe_concurrent.py 1024 1,4 > gpurun_out/concurrent.log 2>&1
