# new tensor-core paths: parity tests, per-layer probe, one ncu --set full capture
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_conv_gpu.py -x -q -k "bf16 or winograd_tc or generic_entry" > gpurun_out/tc_tests.log 2>&1
tail -30 gpurun_out/tc_tests.log
timeout 900 python scripts/probe_tc.py --n 256 --out gpurun_out/probe_tc_resnet.json > gpurun_out/probe_tc_resnet.log 2>&1
cat gpurun_out/probe_tc_resnet.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:igemm_tcgen05 -c 1 -o gpurun_out/ncu_igemm3x_res2 -f python scripts/probe_tc.py --one igemm_3xtf32:64 --layers res2_3x3 --reps 2 > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
