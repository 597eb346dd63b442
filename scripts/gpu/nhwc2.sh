set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "nhwc" > gpurun_out/nhwc_tests.log 2>&1
tail -25 gpurun_out/nhwc_tests.log
timeout 600 python scripts/probe_tc.py --n 256 --kinds direct_nhwc:64,direct_nhwc:128 > gpurun_out/probe_nhwc.log 2>&1
cat gpurun_out/probe_nhwc.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:direct_nhwc -c 1 -o gpurun_out/ncu_nhwc_res4 -f python scripts/probe_tc.py --one direct_nhwc:128 --layers res4_3x3 --reps 2 > gpurun_out/ncu2.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:igemm_pair -c 1 -o gpurun_out/ncu_pair3x_res4 -f python scripts/probe_tc.py --one igemm_3xtf32:256:2 --layers res4_3x3 --reps 2 > gpurun_out/ncu3.log 2>&1
tail -2 gpurun_out/ncu2.log gpurun_out/ncu3.log
