set -x
mkdir -p gpurun_out
TC=direct_nhwc,igemm_3xtf32,igemm_tf32,igemm_bf16,winograd_tc_3xtf32_e2,winograd_tc_3xtf32_e4,winograd_tc_tf32_e4,winograd_tc_bf16_e4
timeout 2400 python scripts/tune_layers.py --workload vgg16 --n 32 --algs $TC > gpurun_out/tune_vgg_tc.log 2>&1
tail -40 gpurun_out/tune_vgg_tc.log
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/b200_vgg16.json
timeout 900 python bench.py --workload vgg16 > gpurun_out/bench_vgg.json 2> gpurun_out/bench_vgg.err
head -c 800 gpurun_out/bench_vgg.json
