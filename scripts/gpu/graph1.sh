set -x
timeout 600 python bench.py > gpurun_out/bench_graph.json 2> gpurun_out/bench_graph.err
head -c 400 gpurun_out/bench_graph.json; tail -5 gpurun_out/bench_graph.err
for N in 32; do timeout 300 python bench.py --batch $N --no-e2e --no-cpu --no-variants > gpurun_out/bench_graph_n$N.json 2> gpurun_out/bench_graph_n$N.err; head -c 300 gpurun_out/bench_graph_n$N.json; done
timeout 900 python -m pytest tests/test_conv_gpu.py -q -x -k "pair or halo or igemm" > gpurun_out/graph_tests.log 2>&1; tail -2 gpurun_out/graph_tests.log
