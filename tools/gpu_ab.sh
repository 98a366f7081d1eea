mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:eval_kernel --launch-skip 943 --launch-count 1 -o gpurun_out/eval0_l16 python tools/probe_bands.py 64 > gpurun_out/ncu_full.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
