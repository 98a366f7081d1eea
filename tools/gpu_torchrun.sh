# bench.py under torchrun (one rank): the launch line the driver uses for N > 1
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/trun.json 2> gpurun_out/trun.err; echo "trun=$?" > gpurun_out/trun_status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 1 --warmup 1 > gpurun_out/trun_ref.json 2> gpurun_out/trun_ref.err; echo "trun_ref=$?" >> gpurun_out/trun_status.txt
