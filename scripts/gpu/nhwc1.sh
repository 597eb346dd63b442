set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_conv_gpu.py -x -q -k "nhwc" > gpurun_out/nhwc_tests.log 2>&1
tail -25 gpurun_out/nhwc_tests.log
timeout 600 python scripts/probe_tc.py --n 256 --kinds direct_nhwc:64,direct_nhwc:128,cudnn_fp32 > gpurun_out/probe_nhwc.log 2>&1
cat gpurun_out/probe_nhwc.log
timeout 600 python bench.py > gpurun_out/bench_pair.json 2> gpurun_out/bench_pair.err
head -c 1500 gpurun_out/bench_pair.json; tail -3 gpurun_out/bench_pair.err
