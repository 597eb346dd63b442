timeout 300 ncu --set full --import-source on --clock-control none -k regex:igemm_pair -s 1 -c 1 -o gpurun_out/ncu_f16gemm2 -f python scripts/f16_one.py res4_3x3 256 3xf16 > /dev/null 2>&1
ls gpurun_out/ncu_f16gemm2*
