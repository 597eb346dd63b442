#!/bin/bash
# ncu evidence for profiles/<ROUND>/ (run through gpurun, one GPU):
#   bash scripts/gpu/evidence.sh [ROUND]
#  1. per tuned layer of ResNet-50 (batch 256) and VGG-16 (batch 32): DRAM bytes and
#     SM<->L2 read bytes per layer call (--cache-control none, last of 3 calls)
#     -> gpurun_out/<ROUND>_{resnet50,vgg16}_traffic.json (bench.py reads them)
#  2. the bench step's kernel launch list (gpu__time_duration, --clock-control none)
#  3. one `ncu --set full` capture of each ResNet-50 layer family's tuned plan, and of the
#     bench's grouped launches of res2 x3 / res4 x5
R=${1:-r2}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum
mkdir -p gpurun_out/traffic_$R
for W in resnet50 vgg16; do
  for L in $(python -c "from paper_2012_15667_b200.runner import WORKLOADS; print(' '.join(s.name for s in WORKLOADS['$W']))"); do
    timeout 300 ncu --metrics $M --cache-control none --print-units base --csv \
      --log-file gpurun_out/traffic_$R/${W}_$L.csv \
      python scripts/run_layer.py --workload $W --layer $L --reps 3 --meta gpurun_out/traffic_$R/${W}_$L.json > /dev/null 2>&1
  done
  python scripts/run_layer.py --workload $W --parse "gpurun_out/traffic_$R/${W}_*.csv" \
    --out gpurun_out/${R}_${W}_traffic.json > /dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-variants --no-cudnn --no-network > gpurun_out/${R}_bench_ncu.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${R}_bench_launches.csv --out gpurun_out/${R}_bench_launches.json > /dev/null
# full captures of the tuned plan of each ResNet-50 layer family (run_layer.py = the bench plan),
# one kernel each (the reports must fit gpurun's 64 MiB return), summarised to JSON
for L in res2_3x3 res3_3x3_s2 res3_3x3 res4_3x3; do
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -s 2 -c 1 \
    -o gpurun_out/${R}_ncu_$L -f python scripts/run_layer.py --workload resnet50 --layer $L --reps 3 > /dev/null 2>&1
done
# the timed step's grouped launches (res2 x3, res4 x5 as one persistent launch each)
for L in res2_3x3 res4_3x3; do
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -s 2 -c 1 \
    -o gpurun_out/${R}_ncu_group_$L -f python scripts/run_layer.py --workload resnet50 --layer $L --group --reps 3 > /dev/null 2>&1
done
python scripts/ncu_summary.py rep gpurun_out/${R}_ncu_*.ncu-rep --out gpurun_out/${R}_ncu_kernels.json > /dev/null 2>&1
rm -rf gpurun_out/traffic_$R/*.csv
# keep one full report (the grouped res4 launch) for reading back; the rest are summarised
find gpurun_out -maxdepth 1 -name "${R}_ncu_*.ncu-rep" ! -name "${R}_ncu_group_res4_3x3.ncu-rep" -delete
ls -la gpurun_out/${R}_*
