set -x
timeout 1200 python scripts/tune_layers.py --workload single --n 1 --algs direct_nhwc,igemm_3xtf32,igemm_tf32,igemm_bf16,winograd_tc_3xtf32_e2,winograd_tc_3xtf32_e4,winograd_tc_tf32_e4,winograd_tc_bf16_e4,winograd_nhwc_e2,winograd_nhwc_e4 > gpurun_out/tune_single.log 2>&1
tail -15 gpurun_out/tune_single.log
cp paper_2012_15667_b200/tuned/b200_single.json gpurun_out/
timeout 300 python bench.py --workload single > gpurun_out/bench_single.json 2> gpurun_out/bench_single.err
head -c 300 gpurun_out/bench_single.json
