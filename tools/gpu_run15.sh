mkdir -p gpurun_out
python tools/probe_align.py 256 > gpurun_out/probe256.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p256.csv python tools/probe_align.py 256 > gpurun_out/ncu_launch.log 2>&1; echo ncu=$? > gpurun_out/status.txt
