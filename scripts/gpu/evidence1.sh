set -x
mkdir -p gpurun_out/traffic2
for L in res2_3x3 res3_3x3_s2 res3_3x3 res4_3x3_s2 res4_3x3 res5_3x3_s2; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/traffic2/resnet50_$L.csv python scripts/run_layer.py --workload resnet50 --layer $L --meta gpurun_out/traffic2/resnet50_$L.json > /dev/null 2>&1
done
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --csv --log-file gpurun_out/traffic2/resnet50_res5_3x3.csv python scripts/run_layer.py --workload resnet50 --layer res5_3x3 --reps 3 --meta gpurun_out/traffic2/resnet50_res5_3x3.json > /dev/null 2>&1
python scripts/run_layer.py --workload resnet50 --parse "gpurun_out/traffic2/resnet50_*.csv" --out gpurun_out/r1_resnet50_traffic.json > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-variants > gpurun_out/b_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/ncu_res3_tsa128 -f python scripts/probe_tc.py --one igemm_3xtf32:128:4 --layers res3_3x3 --reps 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/ncu_res2_fold -f python scripts/probe_tc.py --one igemm_3xtf32:64:2:h32 --layers res2_3x3 --reps 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/ncu_res4_pair256 -f python scripts/probe_tc.py --one igemm_3xtf32:256:2 --layers res4_3x3 --reps 2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
