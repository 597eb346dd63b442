set -x
mkdir -p gpurun_out
timeout 900 python scripts/probe_tc.py --n 256 --kinds direct_nhwc:128,igemm_3xtf32:256:2,igemm_3xtf32:128:1,igemm_tf32:256:2,igemm_bf16:256:2 > gpurun_out/probe_rows.log 2>&1
cat gpurun_out/probe_rows.log
