#!/bin/bash
mkdir -p gpurun_out
for c in c1 c2; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "xc_apply/" --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
  echo "== $c"; python - <<PY
import csv,collections
rows=list(csv.reader(open('gpurun_out/launches_$c.csv')))
hdr=None; agg=collections.OrderedDict()
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if not hdr or len(r)!=len(hdr): continue
    d=dict(zip(hdr,r)); k=d['Kernel Name'][:60]; v=float(d['Metric Value'].replace(',',''))
    a=agg.setdefault(k,[0,0.0]); a[0]+=1; a[1]+=v
for k,(n,t) in agg.items(): print(f"{k:60s} n={n} avg {t/n/1e3:.2f} us")
PY
done
