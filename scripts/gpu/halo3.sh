set -x
for v in 64:2 64:2:h16; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/ncu_res2_tf32_$(echo $v | tr ':' '_') -f python scripts/probe_tc.py --one igemm_tf32:$v --layers res2_3x3 --reps 2 > /dev/null 2>&1
done
ls gpurun_out/*.ncu-rep
