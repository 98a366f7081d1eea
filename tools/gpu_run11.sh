mkdir -p gpurun_out
for i in 1 2 3 4; do python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_r$i.json 2> gpurun_out/bench_r$i.err; done
