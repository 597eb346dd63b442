timeout 600 python -m pytest tests/test_conv_gpu.py tests/test_conv_gpu_fuzz.py -q -x 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -20
timeout 300 python scripts/probe_wtc_chunk.py --layer res3_3x3 --z 128 --nzt 2 --e 4 2>&1 | grep res3
timeout 300 python scripts/probe_wtc_chunk.py --layer res5_3x3 --z 256 --nzt 2 --e 4 2>&1 | grep res5
timeout 600 python scripts/probe_tc.py --n 256 --layers res2_3x3,res3_3x3,res4_3x3,res5_3x3_s2 --kinds igemm_3xtf32:128:2,igemm_3xtf32:256:2 2>&1 | grep res
timeout 300 python bench.py --no-variants 2>&1 | tail -1 > gpurun_out/epi_bench.json
python -c "import json;d=json.load(open('gpurun_out/epi_bench.json'));print(d['value'],d['ms_per_step']);[print(l) for l in d.get('per_layer',[])]"
