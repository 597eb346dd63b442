for cfg in "res3_3x3 128 4 32768" "res4_3x3 256 2 32768" "res5_3x3 256 2 16384"; do set -- $cfg
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max --cache-control none --clock-control none --csv --log-file gpurun_out/wtc10.csv python scripts/probe_wtc_chunk.py --layer $1 --z $2 --nzt $3 --e 4 --one $4 > /dev/null 2>&1
echo "== $cfg"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/wtc10.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ki,ni,vi,ii=H.index('Kernel Name'),H.index('Metric Name'),H.index('Metric Value'),H.index('ID')
d={}
for r in rows[h+1:]:
    if len(r)<=vi: continue
    d.setdefault(int(r[ii]),{'k':r[ki][21:40]})[r[ni]]=r[vi]
for i in sorted(d)[-3:]:
    print(i,d[i])
PY
done
