#!/bin/bash
# per-kernel device times of one sd_attention call at several shapes (ncu launch list)
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/tc_ncu.csv python tools/time_tc.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/tc_ncu.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki,vi,mi,ii=h.index('Kernel Name'),h.index('Metric Value'),h.index('Metric Name'),h.index('ID')
cur={}
for r in rows[hi+1:]:
    if len(r)<=vi: continue
    cur.setdefault(r[ii],{})[r[mi]]=r[vi]; cur[r[ii]]['name']=r[ki][:50]
ids=sorted(cur,key=int)
for i in ids[::23][:40]: print(i, cur[i])
PY
