set -x
TC=igemm_3xtf32,igemm_tf32,igemm_bf16,winograd_tc_3xtf32_e2,winograd_tc_3xtf32_e4,winograd_tc_tf32_e4,winograd_tc_bf16_e4
timeout 1500 python scripts/tune_layers.py --workload resnet50 --n 256 --algs $TC > gpurun_out/tune_resnet_r6.log 2>&1
grep -- "->" gpurun_out/tune_resnet_r6.log
cp paper_2012_15667_b200/tuned/b200_resnet50.json gpurun_out/b200_resnet50.json
timeout 600 python bench.py > gpurun_out/bench_r6.json 2> gpurun_out/bench_r6.err
head -c 300 gpurun_out/bench_r6.json
timeout 1500 python scripts/tune_layers.py --workload vgg16 --n 32 --algs $TC > gpurun_out/tune_vgg_r6.log 2>&1
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/b200_vgg16.json
timeout 900 python bench.py --workload vgg16 > gpurun_out/bench_vgg_r6.json 2> gpurun_out/bench_vgg_r6.err
head -c 300 gpurun_out/bench_vgg_r6.json
