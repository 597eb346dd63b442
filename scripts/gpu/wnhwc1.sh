set -x
timeout 900 python -m pytest tests/test_conv_gpu.py -x -q -k "winograd_tc" > gpurun_out/wnhwc_tests.log 2>&1; tail -15 gpurun_out/wnhwc_tests.log
timeout 1200 python scripts/tune_layers.py --workload resnet50 --n 256 --algs winograd_nhwc_e2,winograd_nhwc_e4 > gpurun_out/tune_wnhwc.log 2>&1
grep "winograd_nhwc" gpurun_out/tune_wnhwc.log
