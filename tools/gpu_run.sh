# One gpurun call: GPU tests, smoke, default bench.  Usage:
#   gpurun --timeout 1500 -- 'bash tools/gpu_run.sh'
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
