set -x
TC=igemm_3xtf32,igemm_tf32,igemm_bf16
timeout 1500 python scripts/tune_layers.py --workload resnet50 --n 256 --algs $TC > gpurun_out/tune_resnet_r9.log 2>&1
grep -- "->" gpurun_out/tune_resnet_r9.log
cp paper_2012_15667_b200/tuned/b200_resnet50.json gpurun_out/b200_resnet50.json
timeout 1500 python scripts/tune_layers.py --workload vgg16 --n 32 --algs $TC > gpurun_out/tune_vgg_r9.log 2>&1
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/b200_vgg16.json
timeout 600 python bench.py > gpurun_out/bench_r9.json 2> gpurun_out/bench_r9.err
timeout 900 python bench.py --workload vgg16 > gpurun_out/bench_vgg_r9.json 2> gpurun_out/bench_vgg_r9.err
head -c 200 gpurun_out/bench_r9.json; head -c 200 gpurun_out/bench_vgg_r9.json
