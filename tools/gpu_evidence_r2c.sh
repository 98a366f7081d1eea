# Round-2 end-of-round evidence (quad expansion kernel) in one box session (writes gpurun_out/ev4/*):
#   gpurun --timeout 3000 -- 'bash tools/gpu_evidence_r2c.sh'
set -u
O=gpurun_out/ev4
mkdir -p $O
timeout 1200 python -m pytest -q -m gpu tests > $O/gpu_tests.log 2>&1; echo "tests=$?" > $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench=$?" >> $O/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref=$?" >> $O/status.txt
timeout 900 python tools/bench_configs.py 3 4 5 > $O/configs.jsonl 2> $O/configs.err; echo "configs=$?" >> $O/status.txt
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --particles 64 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launches=$?" >> $O/status.txt
export BMB_NO_WARMUP=1
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "bmb_band16/" \
  -k regex:"eval_kernel|eval_sub_kernel" --launch-count 2 -o $O/eval_l16 python tools/probe_bands.py 64 > $O/ncu_eval.log 2>&1; echo "ncu_eval=$?" >> $O/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"expand_factored|expand_pair|expand_quad" --launch-skip 1 \
  --launch-count 1 -o $O/expand python tools/probe_bands.py 64 > $O/ncu_exp.log 2>&1; echo "ncu_exp=$?" >> $O/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel \
  --launch-skip 3 --launch-count 1 -o $O/advance python tools/probe_bands.py 1024 > $O/ncu_adv.log 2>&1; echo "ncu_adv=$?" >> $O/status.txt
unset BMB_NO_WARMUP
timeout 900 ncu --set full --clock-control none -k regex:split3_gemm --launch-count 1 -o $O/sweep_gemm \
  python tools/bench_configs.py 4 > $O/ncu_gemm.log 2>&1; echo "ncu_gemm=$?" >> $O/status.txt
timeout 1500 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --csv --log-file $O/step_traffic.csv python tools/step_probe.py 1024 > $O/step_traffic.log 2>&1; echo "traffic=$?" >> $O/status.txt
