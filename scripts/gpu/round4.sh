set -x
mkdir -p gpurun_out/traffic
for L in res2_3x3 res3_3x3_s2 res3_3x3 res4_3x3_s2 res4_3x3 res5_3x3_s2 res5_3x3; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/traffic/resnet50_$L.csv python scripts/run_layer.py --workload resnet50 --layer $L --meta gpurun_out/traffic/resnet50_$L.json > /dev/null 2>&1
done
python scripts/run_layer.py --workload resnet50 --parse "gpurun_out/traffic/resnet50_*.csv" --out gpurun_out/r1_resnet50_traffic.json
mkdir -p profiles; cp gpurun_out/r1_resnet50_traffic.json profiles/
timeout 600 python bench.py > gpurun_out/bench_r4.json 2> gpurun_out/bench_r4.err
head -c 400 gpurun_out/bench_r4.json
TC=direct_nhwc,igemm_3xtf32,igemm_tf32,igemm_bf16,winograd_tc_3xtf32_e2,winograd_tc_3xtf32_e4,winograd_tc_tf32_e4,winograd_tc_bf16_e4
timeout 2400 python scripts/tune_layers.py --workload vgg16 --n 32 --algs $TC > gpurun_out/tune_vgg_tc.log 2>&1
grep -- "->" gpurun_out/tune_vgg_tc.log
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/b200_vgg16.json
timeout 900 python bench.py --workload vgg16 > gpurun_out/bench_vgg.json 2> gpurun_out/bench_vgg.err
head -c 400 gpurun_out/bench_vgg.json
