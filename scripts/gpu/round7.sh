set -x
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "pair" > gpurun_out/r7_tests.log 2>&1; tail -2 gpurun_out/r7_tests.log
timeout 1500 python scripts/tune_layers.py --workload resnet50 --n 256 --algs igemm_3xtf32 > gpurun_out/tune_resnet_r7.log 2>&1
grep -- "->" gpurun_out/tune_resnet_r7.log
cp paper_2012_15667_b200/tuned/b200_resnet50.json gpurun_out/b200_resnet50.json
timeout 1500 python scripts/tune_layers.py --workload vgg16 --n 32 --algs igemm_3xtf32 > gpurun_out/tune_vgg_r7.log 2>&1
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/b200_vgg16.json
timeout 600 python bench.py > gpurun_out/bench_r7.json 2> gpurun_out/bench_r7.err
head -c 300 gpurun_out/bench_r7.json
