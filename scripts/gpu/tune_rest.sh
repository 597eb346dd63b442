mkdir -p gpurun_out
A=igemm_3xtf32,igemm_tf32,igemm_bf16,winograd_tc_3xtf32_e2,winograd_tc_3xtf32_e4,winograd_tc_tf32_e4,winograd_tc_bf16_e4,winograd_nhwc_e2,winograd_nhwc_e4
for n in 128 64 32; do
timeout 1500 python scripts/tune_layers.py --workload resnet50 --n $n --algs $A > gpurun_out/tune_resnet_n$n.log 2>&1
cp paper_2012_15667_b200/tuned/b200_resnet50_n$n.json gpurun_out/
done
timeout 1500 python scripts/tune_layers.py --workload vgg16 --n 32 --algs $A > gpurun_out/tune_vgg16b.log 2>&1
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/
grep -- "->" gpurun_out/tune_vgg16b.log
timeout 600 python bench.py --workload vgg16 > gpurun_out/bench_vgg16b.json 2> gpurun_out/bench_vgg16b.err
python -c "import json;d=json.load(open('gpurun_out/bench_vgg16b.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'])"
for N in 128 64 32; do
  timeout 300 python bench.py --batch $N --no-e2e --no-cpu > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
  head -c 150 gpurun_out/bench_n$N.json; echo
done
