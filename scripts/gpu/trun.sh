timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-variants --no-e2e > gpurun_out/f5_torchrun.json 2> gpurun_out/f5_torchrun.err
wc -l gpurun_out/f5_torchrun.json; head -c 200 gpurun_out/f5_torchrun.json
