mkdir -p gpurun_out
python -m pytest -q -m gpu tests > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
