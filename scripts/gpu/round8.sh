set -x
timeout 1200 python scripts/tune_layers.py --workload resnet50 --n 256 --algs winograd_nhwc_e2,winograd_nhwc_e4 > gpurun_out/tune_wnhwc.log 2>&1
cp paper_2012_15667_b200/tuned/b200_resnet50.json gpurun_out/b200_resnet50.json
timeout 1200 python scripts/tune_layers.py --workload vgg16 --n 32 --algs winograd_nhwc_e2,winograd_nhwc_e4 > gpurun_out/tune_vgg_wnhwc.log 2>&1
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/b200_vgg16.json
timeout 600 python bench.py > gpurun_out/bench_r8.json 2> gpurun_out/bench_r8.err
timeout 900 python bench.py --workload vgg16 > gpurun_out/bench_vgg_r8.json 2> gpurun_out/bench_vgg_r8.err
head -c 200 gpurun_out/bench_r8.json
