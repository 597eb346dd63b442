mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_conv_gpu.py -q -x -k "3xf16" 2>&1 | grep -E "passed|failed" | head -2
 
for n in 256 128 64 32; do
  timeout 900 python scripts/tune_layers.py --workload resnet50 --n $n --algs winograd_tc_3xtf32_e4,winograd_tc_3xf16_e4 > gpurun_out/tune_f16_n$n.log 2>&1
done
timeout 900 python scripts/tune_layers.py --workload vgg16 --n 32 --algs winograd_tc_3xtf32_e4,winograd_tc_3xf16_e4 > gpurun_out/tune_f16_vgg.log 2>&1
cp paper_2012_15667_b200/tuned/*.json gpurun_out/
grep -- "->" gpurun_out/tune_f16_n256.log
timeout 600 python bench.py > gpurun_out/f6_bench.json 2> gpurun_out/f6_bench.err
timeout 600 python bench.py --workload vgg16 > gpurun_out/f6_vgg.json 2> gpurun_out/f6_vgg.err
for N in 128 64 32; do
  timeout 300 python bench.py --batch $N --no-e2e --no-cpu > gpurun_out/f6_n$N.json 2> gpurun_out/f6_n$N.err
done
python -c "
import json
for f in ('f6_bench','f6_vgg','f6_n128','f6_n64','f6_n32'):
    a=json.load(open('gpurun_out/%s.json'%f)); print(f, a['value'], a['ms_per_step'], a['clocks']['reasons'], a['roofline']['frac'])
a=json.load(open('gpurun_out/f6_bench.json'))
for r in a['per_layer']: print(r['layer'], r['algorithm'], r['ms'])"
