timeout 900 python -m pytest tests/test_conv_gpu.py tests/test_conv_gpu_fuzz.py tests/test_graph_replay_gpu.py -q -x 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -5
timeout 300 python scripts/probe_tc.py --n 256 --layers res3_3x3_s2,res4_3x3_s2,res5_3x3_s2 --kinds igemm_3xtf32:128:2,igemm_3xtf32:256:2 2>&1 | grep res
timeout 300 python bench.py --no-variants --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/lo2.json
python -c "import json;a=json.load(open('gpurun_out/lo2.json'));print(a['value'],a['ms_per_step'],a['clocks']['reasons'])"
