set -x
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/splitk_tests.log 2>&1; tail -3 gpurun_out/splitk_tests.log
ALGS=igemm_3xtf32,igemm_tf32,igemm_bf16
for N in 128 64 32; do
  timeout 1200 python scripts/tune_layers.py --workload resnet50 --n $N --algs $ALGS > gpurun_out/tune_resnet_sk_n$N.log 2>&1
  cp paper_2012_15667_b200/tuned/b200_resnet50_n$N.json gpurun_out/
done
for N in 128 64 32; do
  timeout 300 python bench.py --batch $N --no-e2e --no-cpu > gpurun_out/bench_sk_n$N.json 2> gpurun_out/bench_sk_n$N.err
  head -c 150 gpurun_out/bench_sk_n$N.json; echo
done
timeout 600 python bench.py > gpurun_out/bench_r11.json 2> gpurun_out/bench_r11.err
head -c 150 gpurun_out/bench_r11.json
