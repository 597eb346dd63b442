set -x
timeout 900 python -m pytest tests/ -m gpu -q > gpurun_out/f4_tests.log 2>&1; tail -2 gpurun_out/f4_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; tail -1 gpurun_out/f4_smoke.log
timeout 600 python bench.py > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f4_ref.json 2> gpurun_out/f4_ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-variants --no-e2e > gpurun_out/f4_torchrun.json 2> gpurun_out/f4_torchrun.err
timeout 600 python bench.py --workload vgg16 > gpurun_out/f4_vgg.json 2> gpurun_out/f4_vgg.err
timeout 600 python bench.py --workload single > gpurun_out/f4_single.json 2> gpurun_out/f4_single.err
for N in 128 64 32; do
  timeout 300 python bench.py --batch $N --no-e2e --no-cpu > gpurun_out/f4_n$N.json 2> gpurun_out/f4_n$N.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f4_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-variants > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair|winograd_input|winograd_output" -s 3 -c 3 -o gpurun_out/f4_ncu_res4_wino -f python scripts/probe_wtc_chunk.py --layer res4_3x3 --z 256 --nzt 2 --e 4 --one 32768 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/f4_ncu_res3_wino_tsa -s 1 -f python scripts/probe_wtc_chunk.py --layer res3_3x3 --z 128 --nzt 4 --e 4 --one 32768 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/f4_ncu_res5s2_split -f python scripts/probe_tc.py --one igemm_3xtf32:256:2 --layers res5_3x3_s2 --reps 2 > /dev/null 2>&1
python -c "
import json
for f in ('f4_bench','f4_vgg','f4_single','f4_n128','f4_n64','f4_n32','f4_torchrun','f4_ref'):
    a=json.load(open('gpurun_out/%s.json'%f)); print(f, a['value'], a['ms_per_step'], a.get('clocks',{}).get('reasons'), (a.get('roofline') or {}).get('frac'))"
