#!/bin/bash
# pairing slack sweep (XC_PAIR_SLACK): c5, c3, c4
mkdir -p gpurun_out
one() {
  env $2 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline $3 > gpurun_out/exp.json 2> gpurun_out/exp.err || { echo "$1 FAILED"; return; }
  python -c "
import json;d=json.load(open('gpurun_out/exp.json'));r=d['roofline'];print('%-22s'%'$1','ms %.4f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f eff %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac'],r.get('dmma_issue_efficiency',0)))"
}
for v in ${SLACKS:-1.0 1.08 1.2}; do
  for c in c5 c3 c4; do one "$c slack=$v" "XC_PAIR_SLACK=$v" "--config $c"; done
done
