mkdir -p gpurun_out
set -x
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe_fp32_peak.cu -o /tmp/fp32peak && /tmp/fp32peak > gpurun_out/fp32_peak.json
python -m pytest -q -m gpu tests > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
python tools/probe_refine_l16.py 16 > gpurun_out/refine_l16.log 2>&1; echo probe=$? >> gpurun_out/status.txt
python tools/probe_eval.py 16 512 4096 > gpurun_out/sweep16.log 2>&1
python tools/probe_eval.py 24 512 4096 > gpurun_out/sweep24.log 2>&1
cp gpurun_out/fp32_peak.json profiles/fp32_peak.json 2>/dev/null
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
python tools/probe_refine_l16.py 16 > gpurun_out/refine_l16_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 0 -c 2 -o gpurun_out/eval_full python tools/probe_refine_l16.py 16 > gpurun_out/ncu_eval.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
