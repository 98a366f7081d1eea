# ncu counters of every refinement evaluation launch (64-particle band probe)
mkdir -p gpurun_out
timeout 300 python tools/probe_bands.py 64 > gpurun_out/pb64.log 2>&1; echo probe=$? > gpurun_out/status.txt
timeout 1500 ncu --clock-control none -k regex:eval_kernel --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,l1tex__t_bytes.sum --csv --log-file gpurun_out/ncu_eval.csv python tools/probe_bands.py 64 > gpurun_out/ncu_eval.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
