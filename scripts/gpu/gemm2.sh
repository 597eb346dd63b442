set -x
timeout 600 python scripts/probe_gemm.py --m 32768 --n 2048 --k 2048 > gpurun_out/probe_gemm2.log 2>&1
cat gpurun_out/probe_gemm2.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:igemm_pair -c 1 -o gpurun_out/ncu_gemm_tf32_pair256 -f python scripts/probe_gemm.py --m 32768 --n 2048 --k 2048 --one tf32:256:2 > gpurun_out/ncu4.log 2>&1
tail -3 gpurun_out/ncu4.log
