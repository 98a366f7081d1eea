mkdir -p gpurun_out
set -x
python -m pytest -q -m gpu tests -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
BMB_BRICKS=0 python bench.py --no-cpu-baseline > gpurun_out/bench_nobrick.json 2> gpurun_out/bench_nobrick.err
python tools/bench_configs.py 3 4 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo configs=$? >> gpurun_out/status.txt
