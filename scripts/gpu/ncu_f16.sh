timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair|winograd_input|winograd_output" -s 3 -c 3 -o gpurun_out/ncu_res4_f16 -f python scripts/f16_one.py res4_3x3 256 3xf16 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"igemm_pair" -s 1 -c 1 -o gpurun_out/ncu_res2_fold_final -f python scripts/probe_tc.py --one igemm_3xtf32:64:2:h32 --layers res2_3x3 --reps 2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep | tail -3
