set -x
timeout 600 python bench.py > gpurun_out/bench_r12.json 2> gpurun_out/bench_r12.err
timeout 900 python bench.py --workload vgg16 > gpurun_out/bench_vgg_r12.json 2> gpurun_out/bench_vgg_r12.err
timeout 300 python bench.py --workload single > gpurun_out/bench_single_r12.json 2> gpurun_out/bench_single_r12.err
for N in 128 64 32; do timeout 300 python bench.py --batch $N --no-e2e --no-cpu > gpurun_out/bench_r12_n$N.json 2> gpurun_out/bench_r12_n$N.err; done
for f in gpurun_out/bench_r12.json gpurun_out/bench_vgg_r12.json gpurun_out/bench_single_r12.json gpurun_out/bench_r12_n*.json; do head -c 160 $f; echo; done
