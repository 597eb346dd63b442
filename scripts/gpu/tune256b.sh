mkdir -p gpurun_out
A=igemm_3xtf32,igemm_tf32,igemm_bf16,winograd_tc_3xtf32_e2,winograd_tc_3xtf32_e4,winograd_tc_tf32_e4,winograd_tc_bf16_e4,winograd_nhwc_e2,winograd_nhwc_e4
timeout 3000 python scripts/tune_layers.py --workload resnet50 --n 256 --algs $A > gpurun_out/tune_resnet256b.log 2>&1
grep -- "->" gpurun_out/tune_resnet256b.log
cp paper_2012_15667_b200/tuned/b200_resnet50.json gpurun_out/b200_resnet50.json
timeout 600 python bench.py > gpurun_out/bench_t256b.json 2> gpurun_out/bench_t256b.err
python -c "import json;d=json.load(open('gpurun_out/bench_t256b.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline'],d.get('variants'))"
