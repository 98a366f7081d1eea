mkdir -p gpurun_out
set -x
python -m pytest -q -m gpu tests -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
python tools/probe_align.py 128 > gpurun_out/probe_align.log 2>&1; echo probe=$? >> gpurun_out/status.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
python bench.py --expand gemm --no-cpu-baseline > gpurun_out/bench_gemm.json 2> gpurun_out/bench_gemm.err; echo bench_gemm=$? >> gpurun_out/status.txt
