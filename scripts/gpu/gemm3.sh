timeout 600 python scripts/probe_gemm.py --m 32768 --n 2048 --k 2048 2>&1 | grep -v "^$"
