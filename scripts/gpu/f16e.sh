timeout 600 python -m pytest tests/test_conv_gpu.py -q -x -k "3xf16" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -5
timeout 600 python scripts/f16_check.py 2>&1 | grep -E "ms|err" | tail -18
timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/f16e.csv python scripts/f16_one.py res4_3x3 256 3xf16 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/f16e.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ki,vi=H.index('Kernel Name'),H.index('Metric Value')
for r in rows[h+1:][-3:]: print(r[ki][:60], r[vi])
PY
