timeout 900 python -m pytest tests/ -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_f3.json 2> gpurun_out/bench_f3.err
timeout 600 python bench.py --workload vgg16 > gpurun_out/bench_f3vgg.json 2> gpurun_out/bench_f3vgg.err
for N in 128 64 32; do
  timeout 300 python bench.py --batch $N --no-e2e --no-cpu > gpurun_out/bench_f3_n$N.json 2> gpurun_out/bench_f3_n$N.err
done
python -c "
import json
for f in ('bench_f3','bench_f3vgg','bench_f3_n128','bench_f3_n64','bench_f3_n32'):
    a=json.load(open('gpurun_out/%s.json'%f)); print(f, a['value'], a['ms_per_step'], a['clocks']['reasons'], a['roofline']['frac'])"
