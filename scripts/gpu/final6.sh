timeout 900 python -m pytest tests/ -m gpu -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f7_ref.json 2>/dev/null
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-variants --no-e2e > gpurun_out/f7_torchrun.json 2> gpurun_out/f7_torchrun.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f7_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
wc -l gpurun_out/f7_torchrun.json
