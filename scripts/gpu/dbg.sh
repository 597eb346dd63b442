for v in 3xtf32:128:2 3xtf32:256:2 tf32:128:2; do echo "== $v"; timeout 300 python scripts/probe_gemm.py --m 32768 --n 2048 --k 2048 --one $v 2>&1 | grep "MMA thread" | head -2; done
