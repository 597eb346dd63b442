timeout 900 python -m pytest tests/test_device_api_gpu.py -q -p no:cacheprovider 2>&1 | tail -5
mkdir -p gpurun_out/tuned2
cp paper_2012_15667_b200/tuned/b200_resnet50.json gpurun_out/tuned2/
timeout 1200 python scripts/tune_layers.py --workload resnet50 --n 256 --algs igemm_3xf16,winograd_tc_3xf16_e4 --out gpurun_out/tuned2/b200_resnet50.json 2>&1 | grep -e "->\|configs" | tail -30
