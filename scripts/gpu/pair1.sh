set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "igemm or winograd_tc" > gpurun_out/pair_tests.log 2>&1
tail -25 gpurun_out/pair_tests.log
timeout 900 python scripts/probe_tc.py --n 256 --kinds igemm_3xtf32:128,igemm_3xtf32:256,igemm_tf32:128,igemm_tf32:256,igemm_bf16:256,winograd_tc_3xtf32:4:256,winograd_tc_tf32:4:256,cudnn_tf32 --out gpurun_out/probe_pair.json > gpurun_out/probe_pair.log 2>&1
cat gpurun_out/probe_pair.log
