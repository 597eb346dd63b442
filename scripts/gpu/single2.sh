timeout 600 python bench.py --workload single > gpurun_out/bench_single2.json 2> gpurun_out/bench_single2.err
python -c "
import json;a=json.load(open('gpurun_out/bench_single2.json'));print(a['value'],a['ms_per_step'],a['config'],a['roofline']['frac'],a.get('variants',{}).keys())
for r in a['per_layer']: print(r)"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref2.json 2>/dev/null; head -c 250 gpurun_out/bench_ref2.json
