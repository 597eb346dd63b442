set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "igemm or winograd_tc" > gpurun_out/pair2_tests.log 2>&1
tail -5 gpurun_out/pair2_tests.log
TC=igemm_3xtf32,igemm_tf32,igemm_bf16,winograd_tc_3xtf32_e2,winograd_tc_3xtf32_e4,winograd_tc_tf32_e4,winograd_tc_bf16_e4
timeout 1500 python scripts/tune_layers.py --workload resnet50 --n 64 --algs $TC > gpurun_out/tune_resnet_tc.log 2>&1
tail -40 gpurun_out/tune_resnet_tc.log
cp paper_2012_15667_b200/tuned/b200_resnet50.json gpurun_out/
timeout 600 python bench.py > gpurun_out/bench_pair.json 2> gpurun_out/bench_pair.err
head -c 1500 gpurun_out/bench_pair.json
