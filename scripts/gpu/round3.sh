set -x
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -5 gpurun_out/gpu_tests.log
TC=igemm_3xtf32,igemm_tf32,igemm_bf16
timeout 1200 python scripts/tune_layers.py --workload resnet50 --n 256 --algs $TC > gpurun_out/tune_resnet_tc3.log 2>&1
grep -- "->" gpurun_out/tune_resnet_tc3.log
cp paper_2012_15667_b200/tuned/b200_resnet50.json gpurun_out/b200_resnet50.json
timeout 600 python bench.py > gpurun_out/bench_r3.json 2> gpurun_out/bench_r3.err
head -c 600 gpurun_out/bench_r3.json
