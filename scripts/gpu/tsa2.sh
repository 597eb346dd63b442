set -x
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -c 1 -o gpurun_out/ncu_res2_tsa64 -f python scripts/probe_tc.py --one igemm_3xtf32:64:4 --layers res2_3x3 --reps 2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
