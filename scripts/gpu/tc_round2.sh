set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -15 gpurun_out/gpu_tests.log
timeout 900 python scripts/probe_tc.py --n 256 --kinds igemm_3xtf32:64,igemm_3xtf32:128,igemm_3xtf32:256,winograd_tc_3xtf32:4:128,winograd_tc_3xtf32:4:256,winograd_tc_3xtf32:2:256 --out gpurun_out/probe_tc2.json > gpurun_out/probe_tc2.log 2>&1
cat gpurun_out/probe_tc2.log
