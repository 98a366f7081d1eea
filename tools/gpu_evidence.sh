# Round evidence: GPU tests, smoke, bench (both arms), launch list, ncu --set full of the top kernels.
#   gpurun --timeout 3000 -- 'bash tools/gpu_evidence.sh'
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$? >> gpurun_out/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --particles 64 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$? >> gpurun_out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:eval_kernel --launch-skip 942 --launch-count 2 -o gpurun_out/eval_l16 python tools/probe_bands.py 64 > gpurun_out/ncu_eval.log 2>&1; echo ncu_eval=$? >> gpurun_out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:expand_factored --launch-skip 1 --launch-count 1 -o gpurun_out/expand_l16 python tools/probe_bands.py 64 > gpurun_out/ncu_exp.log 2>&1; echo ncu_exp=$? >> gpurun_out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:compose_kernel --launch-skip 23 --launch-count 1 -o gpurun_out/compose_l16 python tools/probe_bands.py 64 > gpurun_out/ncu_comp.log 2>&1; echo ncu_comp=$? >> gpurun_out/status.txt
