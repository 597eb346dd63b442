set -x
mkdir -p gpurun_out/traffic3 gpurun_out/traffic_vgg3
for L in res2_3x3 res3_3x3_s2 res4_3x3_s2 res5_3x3_s2; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/traffic3/resnet50_$L.csv python scripts/run_layer.py --workload resnet50 --layer $L --meta gpurun_out/traffic3/resnet50_$L.json > /dev/null 2>&1
done
for L in res3_3x3 res4_3x3 res5_3x3; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --csv --log-file gpurun_out/traffic3/resnet50_$L.csv python scripts/run_layer.py --workload resnet50 --layer $L --reps 3 --meta gpurun_out/traffic3/resnet50_$L.json > /dev/null 2>&1
done
python scripts/run_layer.py --workload resnet50 --parse "gpurun_out/traffic3/resnet50_*.csv" --out gpurun_out/r1_resnet50_traffic.json > /dev/null
for L in conv1_1 conv1_2 conv2_1 conv2_2 conv3_1 conv3_2 conv4_1 conv4_2 conv5_1; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --csv --log-file gpurun_out/traffic_vgg3/vgg16_$L.csv python scripts/run_layer.py --workload vgg16 --layer $L --reps 3 --meta gpurun_out/traffic_vgg3/vgg16_$L.json > /dev/null 2>&1
done
python scripts/run_layer.py --workload vgg16 --parse "gpurun_out/traffic_vgg3/vgg16_*.csv" --out gpurun_out/r1_vgg16_traffic.json > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-variants > gpurun_out/b_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair|winograd_input|winograd_output" -s 3 -c 3 -o gpurun_out/ncu_res4_wino -f python scripts/probe_wtc_chunk.py --layer res4_3x3 --z 256 --nzt 2 --e 4 --one 32768 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/ncu_res2_fold -f python scripts/probe_tc.py --one igemm_3xtf32:64:2:h32 --layers res2_3x3 --reps 2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
