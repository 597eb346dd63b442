mkdir -p gpurun_out/tuned
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/tuned/
timeout 900 python scripts/tune_layers.py --workload vgg16 --n 32 --algs igemm_3xf16 --out gpurun_out/tuned/b200_vgg16.json 2>&1 | grep -e "->" | tail -20
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/r2h_bench.log 2>&1; tail -c 1500 gpurun_out/r2h_bench.log
