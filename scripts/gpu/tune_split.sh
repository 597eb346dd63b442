mkdir -p gpurun_out
A=igemm_3xtf32,igemm_tf32,igemm_bf16
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x -k "split or pair" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -5
for n in 256 128 64 32; do
  timeout 1500 python scripts/tune_layers.py --workload resnet50 --n $n --algs $A > gpurun_out/tune_split_n$n.log 2>&1
done
cp paper_2012_15667_b200/tuned/b200_resnet50*.json gpurun_out/
timeout 1500 python scripts/tune_layers.py --workload vgg16 --n 32 --algs $A > gpurun_out/tune_split_vgg.log 2>&1
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/
timeout 600 python bench.py > gpurun_out/bench_split256.json 2> gpurun_out/bench_split256.err
timeout 600 python bench.py --workload vgg16 > gpurun_out/bench_splitvgg.json 2> gpurun_out/bench_splitvgg.err
for N in 128 64 32; do
  timeout 300 python bench.py --batch $N --no-e2e --no-cpu > gpurun_out/bench_split_n$N.json 2> gpurun_out/bench_split_n$N.err
done
python -c "
import json
for f in ('bench_split256','bench_splitvgg','bench_split_n128','bench_split_n64','bench_split_n32'):
    a=json.load(open('gpurun_out/%s.json'%f)); print(f, a['value'], a['ms_per_step'], a.get('e2e',{}).get('value'), a['roofline']['frac'])"
