mkdir -p gpurun_out
for i in 1 2 3; do python bench.py --no-cpu-baseline > gpurun_out/bench_r$i.json 2> gpurun_out/bench_r$i.err; done
python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_s10.json 2> gpurun_out/bench_s10.err
