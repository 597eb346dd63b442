set -x
timeout 600 python scripts/probe_gemm.py > gpurun_out/probe_gemm.log 2>&1
timeout 600 python scripts/probe_gemm.py --m 32768 --n 2048 --k 2048 >> gpurun_out/probe_gemm.log 2>&1
cat gpurun_out/probe_gemm.log
