mkdir -p gpurun_out
python -m pytest -q -m gpu tests > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
python tools/bench_configs.py 5 > gpurun_out/cfg5.jsonl 2> gpurun_out/cfg5.err; echo cfg5=$? >> gpurun_out/status.txt
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo torchrun=$? >> gpurun_out/status.txt
