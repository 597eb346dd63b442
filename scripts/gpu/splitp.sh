timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | grep -E "^E  |FAILED|passed|failed" | head
timeout 300 python scripts/probe_tc.py --n 256 --layers res3_3x3_s2,res4_3x3_s2,res5_3x3_s2 --kinds igemm_3xtf32:128:2,igemm_3xtf32:256:2 2>&1 | grep res
timeout 300 python bench.py --no-variants --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/sp256.json
timeout 300 python bench.py --batch 32 --no-variants --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/sp32.json
timeout 300 python bench.py --batch 64 --no-variants --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/sp64.json
python -c "
import json
for f in ('sp256','sp64','sp32'):
    a=json.load(open('gpurun_out/%s.json'%f)); print(f, a['value'], a['ms_per_step'], [(r['layer'],r['ms']) for r in a['per_layer'] if 's2' in r['layer']])"
