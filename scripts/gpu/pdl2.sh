cp paper_2012_15667_b200/lib/exp/libexp.so paper_2012_15667_b200/lib/libconvio_b200.so
for pdl in 0 1 0 1; do
  CONVIO_PDL=$pdl timeout 300 python bench.py --no-variants --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/pdl_$pdl.json
  CONVIO_PDL=$pdl timeout 300 python bench.py --batch 32 --no-variants --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/pdl32_$pdl.json
  python -c "import json;a=json.load(open('gpurun_out/pdl_$pdl.json'));b=json.load(open('gpurun_out/pdl32_$pdl.json'));print('no-trigger PDL=$pdl', a['value'], a['ms_per_step'], b['value'], b['ms_per_step'])"
done
