timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:"igemm_pair|winograd_input_tc|winograd_output_tc" -s 3 -c 3 -o gpurun_out/wtc_res3b python scripts/probe_wtc_chunk.py --layer res3_3x3 --z 128 --nzt 2 --e 4 --one 16384 > gpurun_out/wtc4.log 2>&1
tail -3 gpurun_out/wtc4.log
