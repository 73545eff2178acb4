#!/bin/bash
# c1 small path: kernel durations and instruction counts (ncu), plus the bench line
mkdir -p gpurun_out
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c1.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/c1.json'));r=d['roofline'];print('c1 ms %.4f'%d['ms_per_step'],'eager %.4f'%d['graph']['eager_ms_per_step'],'spmm %.4f fft %.4f'%(r['spmm_ms'],r['fft_ms']))"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_active.max,smsp__pcsamp_warps_issue_stalled_no_instructions,launch__grid_size --clock-control none --cache-control none --nvtx --nvtx-include "xc_apply/" --csv --log-file gpurun_out/launches_c1.csv python bench.py --config c1 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python - <<PY
import csv,collections
rows=list(csv.reader(open('gpurun_out/launches_c1.csv')))
hdr=None; agg=collections.OrderedDict()
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if not hdr or len(r)!=len(hdr): continue
    d=dict(zip(hdr,r)); k=(d['Kernel Name'][:50], d['Metric Name']); v=float(d['Metric Value'].replace(',',''))
    a=agg.setdefault(k,[0,0.0]); a[0]+=1; a[1]+=v
for (k,m),(n,t) in agg.items(): print(f"{k:50s} {m:32s} n={n} avg {t/n:.1f}")
PY
