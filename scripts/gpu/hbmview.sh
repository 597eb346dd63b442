timeout 600 python bench.py --no-variants --no-e2e 2>/dev/null | tail -1 > gpurun_out/hv.json
python -c "import json;a=json.load(open('gpurun_out/hv.json'));print(a['value'], a['roofline'])"
