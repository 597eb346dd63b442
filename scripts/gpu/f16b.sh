timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/f16b.csv python scripts/f16_one.py res4_3x3 256 3xf16 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/f16b.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ki,vi=H.index('Kernel Name'),H.index('Metric Value')
for r in rows[h+1:][-4:]: print(r[ki][:60], r[vi])
PY


timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/f16c.csv python scripts/f16_one.py res3_3x3 128 3xf16 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/f16c.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ki,vi=H.index('Kernel Name'),H.index('Metric Value')
for r in rows[h+1:][-4:]: print(r[ki][:60], r[vi])
PY
