mkdir -p gpurun_out
set -x
python -m pytest -q -m gpu tests > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
for k in 1 2 4; do BMB_SWEEP_K=$k python tools/probe_eval.py 16 512 4096 > gpurun_out/sweep16_k$k.log 2>&1; BMB_SWEEP_K=$k python tools/probe_eval.py 24 512 4096 > gpurun_out/sweep24_k$k.log 2>&1; done
for k in 1 0; do BMB_EVAL_K=$k python tools/probe_refine_l16.py 16 > gpurun_out/refine_l16_k$k.log 2>&1; done
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
BMB_EVAL_K=1 python bench.py --no-cpu-baseline > gpurun_out/bench_k1.json 2> gpurun_out/bench_k1.err
BMB_SWEEP_K=1 python tools/probe_eval.py 16 512 4096 > /dev/null 2>&1 && \
BMB_SWEEP_K=1 ncu --set full --clock-control none --import-source on -k regex:eval_sweep -s 1 -c 1 -o gpurun_out/sweep_k1 python tools/probe_eval.py 16 512 4096 > gpurun_out/ncu_sweep.log 2>&1
BMB_SWEEP_K=4 python tools/probe_eval.py 16 512 4096 > /dev/null 2>&1 && \
BMB_SWEEP_K=4 ncu --set full --clock-control none --import-source on -k regex:eval_sweep -s 1 -c 1 -o gpurun_out/sweep_k4 python tools/probe_eval.py 16 512 4096 >> gpurun_out/ncu_sweep.log 2>&1
echo ncu=$? >> gpurun_out/status.txt
