mkdir -p gpurun_out/tr_f16r gpurun_out/tr_f16v
for L in res4_3x3 res5_3x3; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --csv --log-file gpurun_out/tr_f16r/resnet50_$L.csv python scripts/run_layer.py --workload resnet50 --layer $L --reps 3 --meta gpurun_out/tr_f16r/resnet50_$L.json > /dev/null 2>&1
done
python scripts/run_layer.py --workload resnet50 --parse gpurun_out/tr_f16r/resnet50_*.csv --out gpurun_out/tr_f16_resnet50.json > /dev/null
for L in conv3_2 conv4_1 conv4_2 conv5_1; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --csv --log-file gpurun_out/tr_f16v/vgg16_$L.csv python scripts/run_layer.py --workload vgg16 --layer $L --reps 3 --meta gpurun_out/tr_f16v/vgg16_$L.json > /dev/null 2>&1
done
python scripts/run_layer.py --workload vgg16 --parse gpurun_out/tr_f16v/vgg16_*.csv --out gpurun_out/tr_f16_vgg16.json > /dev/null
cat gpurun_out/tr_f16_resnet50.json | head -30
