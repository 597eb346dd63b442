for cfg in "res4_3x3 256 2 32768" "res3_3x3 128 4 32768"; do set -- $cfg
timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/wib.csv python scripts/probe_wtc_chunk.py --layer $1 --z $2 --nzt $3 --e 4 --one $4 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/wib.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ki,vi=H.index('Kernel Name'),H.index('Metric Value')
print([ (r[ki][21:45], r[vi]) for r in rows[h+1:] if 'input' in r[ki]][-2:])
PY
timeout 300 python scripts/probe_wtc_chunk.py --layer $1 --z $2 --nzt $3 --e 4 --sweep $4 2>&1 | grep res
done
