mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/tc_ncu.csv python tools/time_tc.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/tc_ncu.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki,vi,mi,ii=h.index('Kernel Name'),h.index('Metric Value'),h.index('Metric Name'),h.index('ID')
cur=collections.OrderedDict()
for r in rows[hi+1:]:
    if len(r)<=vi: continue
    d=cur.setdefault(r[ii],{}); d[r[mi]]=r[vi]; d['name']=r[ki][:40]
ids=list(cur)
# time_tc: 4 shapes x (3 warm + 20 timed) calls x (tc + merge) kernels
per=len(ids)//4
for s in range(4):
    blk=[cur[i] for i in ids[s*per:(s+1)*per]]
    agg=collections.defaultdict(list)
    for d in blk: agg[d['name']].append(float(d['gpu__time_duration.sum']))
    print('shape',s, {k:(len(v), round(sorted(v)[len(v)//2],1)) for k,v in agg.items()})
PY
