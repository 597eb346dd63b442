set -x
./scripts/dev/umma_shift_selftest > gpurun_out/umma_shift.log 2>&1; tail -8 gpurun_out/umma_shift.log
timeout 600 python bench.py --workload single > gpurun_out/bench_single.json 2> gpurun_out/bench_single.err
head -c 1500 gpurun_out/bench_single.json; tail -3 gpurun_out/bench_single.err
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --csv --log-file gpurun_out/traffic/resnet50_res5_3x3_warm.csv python scripts/run_layer.py --workload resnet50 --layer res5_3x3 --reps 3 --meta gpurun_out/traffic/resnet50_res5_3x3_warm.json > /dev/null 2>&1
python scripts/run_layer.py --workload resnet50 --parse "gpurun_out/traffic/resnet50_res5_3x3_warm.csv" --out gpurun_out/r1_resnet50_res5_warm_traffic.json
