set -x
ALGS=direct_nhwc,igemm_3xtf32,igemm_tf32,igemm_bf16,winograd_tc_3xtf32_e4,winograd_tc_tf32_e4,winograd_tc_bf16_e4,winograd_nhwc_e4
for N in 128 64 32; do
  timeout 1200 python scripts/tune_layers.py --workload resnet50 --n $N --algs $ALGS > gpurun_out/tune_resnet_n$N.log 2>&1
  cp paper_2012_15667_b200/tuned/b200_resnet50_n$N.json gpurun_out/
  grep -- "->" gpurun_out/tune_resnet_n$N.log | head -3
done
for N in 128 64 32; do
  timeout 300 python bench.py --batch $N --no-e2e --no-cpu > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
  head -c 150 gpurun_out/bench_n$N.json; echo
done
