for pdl in 1 0 1 0; do
  CONVIO_PDL=$pdl timeout 300 python bench.py --workload vgg16 --no-variants --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/pv.json
  python -c "import json;a=json.load(open('gpurun_out/pv.json'));print('PDL=$pdl', a['value'], a['ms_per_step'], a['clocks']['reasons'], [(r['layer'],r['ms']) for r in a['per_layer'][:3]])"
done
