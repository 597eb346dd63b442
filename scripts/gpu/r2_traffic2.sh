M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum
mkdir -p gpurun_out/traffic2
for L in res2_3x3 res3_3x3_s2 res4_3x3_s2 res5_3x3_s2 res4_3x3; do
  timeout 300 ncu --metrics $M --cache-control none --print-units base --csv --log-file gpurun_out/traffic2/resnet50_$L.csv \
      python scripts/run_layer.py --workload resnet50 --layer $L --reps 3 --meta gpurun_out/traffic2/resnet50_$L.json > /dev/null 2>&1
done
python scripts/run_layer.py --workload resnet50 --parse "gpurun_out/traffic2/resnet50_*.csv" --out gpurun_out/r2_traffic2.json > /dev/null
timeout 300 python scripts/probe_tc.py --n 256 --kinds igemm_3xf16:64:2:h32,igemm_3xf16:128:2,igemm_3xf16:256:2 --reps 10 2>&1 | grep " ms"
