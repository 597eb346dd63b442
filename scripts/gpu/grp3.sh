timeout 600 python -m pytest tests/test_conv_gpu.py tests/test_conv_gpu_fuzz.py -q -x -k "pair or halo or igemm or randomized" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -20
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/grp_bench.json
python -c "import json;d=json.load(open('gpurun_out/grp_bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'])"
