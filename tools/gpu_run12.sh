mkdir -p gpurun_out
python -m pytest -q -m gpu tests -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
for i in 1 2; do python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_r$i.json 2> gpurun_out/bench_r$i.err; done
