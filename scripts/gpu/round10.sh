set -x
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "winograd_tc" > gpurun_out/r10_tests.log 2>&1; tail -2 gpurun_out/r10_tests.log
W=winograd_tc_3xtf32_e4,winograd_tc_3xtf32_e2,winograd_tc_tf32_e4,winograd_tc_bf16_e4,winograd_nhwc_e4,winograd_nhwc_e2
timeout 1500 python scripts/tune_layers.py --workload resnet50 --n 256 --algs $W > gpurun_out/tune_resnet_r10.log 2>&1
grep -E "winograd|->" gpurun_out/tune_resnet_r10.log | tail -12
cp paper_2012_15667_b200/tuned/b200_resnet50.json gpurun_out/b200_resnet50.json
timeout 1500 python scripts/tune_layers.py --workload vgg16 --n 32 --algs $W > gpurun_out/tune_vgg_r10.log 2>&1
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/b200_vgg16.json
timeout 600 python bench.py > gpurun_out/bench_r10.json 2> gpurun_out/bench_r10.err
timeout 900 python bench.py --workload vgg16 > gpurun_out/bench_vgg_r10.json 2> gpurun_out/bench_vgg_r10.err
head -c 200 gpurun_out/bench_r10.json; head -c 200 gpurun_out/bench_vgg_r10.json
