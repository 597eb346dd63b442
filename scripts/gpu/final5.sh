timeout 900 python -m pytest tests/ -m gpu -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/f5_bench.json 2> gpurun_out/f5_bench.err
timeout 600 python bench.py --workload vgg16 > gpurun_out/f5_vgg.json 2> gpurun_out/f5_vgg.err
python -c "
import json
for f in ('f5_bench','f5_vgg'):
    a=json.load(open('gpurun_out/%s.json'%f)); print(f, a['value'], a['ms_per_step'], a['clocks']['reasons'], a['roofline']['frac'], a['e2e']['value'])"
