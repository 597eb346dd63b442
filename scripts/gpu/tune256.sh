set -x
mkdir -p gpurun_out
timeout 3000 python scripts/tune_layers.py --workload resnet50 --n 256 > gpurun_out/tune_resnet256.log 2>&1
tail -60 gpurun_out/tune_resnet256.log
cp paper_2012_15667_b200/tuned/b200_resnet50.json gpurun_out/b200_resnet50.json
timeout 600 python bench.py > gpurun_out/bench_t256.json 2> gpurun_out/bench_t256.err
head -c 1200 gpurun_out/bench_t256.json
