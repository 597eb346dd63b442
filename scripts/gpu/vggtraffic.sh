mkdir -p gpurun_out/traffic_vgg
for L in conv1_1 conv1_2 conv2_1 conv2_2 conv3_1 conv3_2 conv4_1 conv4_2 conv5_1; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --csv --log-file gpurun_out/traffic_vgg/vgg16_$L.csv python scripts/run_layer.py --workload vgg16 --layer $L --reps 3 --meta gpurun_out/traffic_vgg/vgg16_$L.json > /dev/null 2>&1
done
python scripts/run_layer.py --workload vgg16 --parse "gpurun_out/traffic_vgg/vgg16_*.csv" --out gpurun_out/r1_vgg16_traffic.json | head -5
