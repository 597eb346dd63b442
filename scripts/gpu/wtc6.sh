timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/wtc6_launches.csv python scripts/probe_wtc_chunk.py --layer res3_3x3 --z 128 --nzt 2 --e 4 --one 16384 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/wtc6_launches.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ki,ni,vi,ii=H.index('Kernel Name'),H.index('Metric Name'),H.index('Metric Value'),H.index('ID')
d={}
for r in rows[h+1:]:
    if len(r)<=vi: continue
    d.setdefault(int(r[ii]),{'k':r[ki][:40]})[r[ni]]=r[vi]
for i in sorted(d)[-6:]:
    print(i,d[i])
PY
for L in res2_3x3:64 res4_3x3:256; do l=${L%%:*}; z=${L##*:}; timeout 300 python scripts/probe_wtc_chunk.py --layer $l --z $z --nzt 2 --e 4 2>&1 | grep res; done
