timeout 600 python bench.py > gpurun_out/f8_bench.json 2> gpurun_out/f8_bench.err
timeout 600 python bench.py --workload vgg16 > gpurun_out/f8_vgg.json 2> gpurun_out/f8_vgg.err
python -c "
import json
for f in ('f8_bench','f8_vgg'):
    a=json.load(open('gpurun_out/%s.json'%f)); r=a['roofline']; print(f, a['value'], a['ms_per_step'], a['clocks']['reasons'], r['kernel'][:40], r['frac'], r.get('hbm_view',{}).get('frac'), r['share_of_step'])"
