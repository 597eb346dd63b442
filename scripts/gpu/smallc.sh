timeout 600 python -m pytest tests/test_conv_gpu.py -q -x -k "small_c or direct" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -5
timeout 900 python scripts/tune_layers.py --workload vgg16 --n 32 --algs direct_nhwc --layers conv1_1 2>&1 | grep -E "direct_nhwc|->"
cp paper_2012_15667_b200/tuned/b200_vgg16.json gpurun_out/b200_vgg16.json
timeout 600 python bench.py --workload vgg16 --no-e2e --no-variants 2>/dev/null | tail -1 > gpurun_out/vsc.json
python -c "import json;a=json.load(open('gpurun_out/vsc.json'));print(a['value'],a['ms_per_step']);print([(r['layer'],r['algorithm'],r['ms']) for r in a['per_layer'][:2]])"
