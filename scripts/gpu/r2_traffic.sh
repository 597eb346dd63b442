# per-layer ncu: DRAM bytes and SM<->L2 read bytes per tuned layer call (cache-control none, 3 calls)
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum
mkdir -p gpurun_out/traffic
for W in resnet50 vgg16; do
  for L in $(python -c "from paper_2012_15667_b200.runner import WORKLOADS; print(' '.join(s.name for s in WORKLOADS['$W']))"); do
    timeout 300 ncu --metrics $M --cache-control none --print-units base --csv --log-file gpurun_out/traffic/${W}_$L.csv \
      python scripts/run_layer.py --workload $W --layer $L --reps 3 --meta gpurun_out/traffic/${W}_$L.json > /dev/null 2>&1
  done
  python scripts/run_layer.py --workload $W --parse "gpurun_out/traffic/${W}_*.csv" --out gpurun_out/r2_${W}_traffic.json > /dev/null
done
ls gpurun_out/traffic | head -50
