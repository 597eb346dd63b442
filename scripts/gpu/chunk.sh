python scripts/probe_wtc_chunk.py --workload resnet50 --layer res5_3x3 --n 256 2>&1 | grep s_b
python scripts/probe_wtc_chunk.py --workload vgg16 --layer conv4_2 --n 32 2>&1 | grep s_b
python scripts/probe_wtc_chunk.py --workload vgg16 --layer conv3_2 --n 32 2>&1 | grep s_b
for SB in 1024 4096 16384; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --csv --log-file gpurun_out/chunk_$SB.csv python scripts/probe_wtc_chunk.py --workload resnet50 --layer res5_3x3 --n 256 --one $SB > /dev/null 2>&1
  python - $SB <<'PY'
import csv,sys
rows=list(csv.reader(open(f"gpurun_out/chunk_{sys.argv[1]}.csv")))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); ni=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
per={}
for r in rows[hdr+1:]:
    if 'convio' not in r[ki] or 'filter' in r[ki]: continue
    per.setdefault(int(r[ii]),0.0); per[int(r[ii])]+=float(r[vi].replace(',',''))
ids=sorted(per); last=ids[-len(ids)//3:]
print("s_b", sys.argv[1], "DRAM MB per call", round(sum(per[i] for i in last)/1e6,1), "kernels", len(last))
PY
done
