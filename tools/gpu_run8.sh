mkdir -p gpurun_out
set -x
python -m pytest -q -m gpu tests -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
python tools/probe_refine_l16.py 16 > gpurun_out/refine_l16.log 2>&1
python tools/bench_configs.py 4 > gpurun_out/configs4.jsonl 2>&1
