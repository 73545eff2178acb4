#!/bin/bash
# env sweep: PF instance and items per window (c3, c4, c5)
mkdir -p gpurun_out
one() {
  env $2 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline $3 > gpurun_out/exp.json 2> gpurun_out/exp.err || { echo "$1 FAILED"; return; }
  python -c "
import json;d=json.load(open('gpurun_out/exp.json'));r=d['roofline'];print('%-22s'%'$1','ms %.4f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac']))"
}
for c in c3 c4; do
  one "$c default" "XC_X=0" "--config $c"
  one "$c PF=0" "XC_SPMM_PF=0" "--config $c"
  one "$c PF=1" "XC_SPMM_PF=1" "--config $c"
  one "$c items32" "XC_WIN_ITEMS_A=32" "--config $c"
  one "$c items48" "XC_WIN_ITEMS_A=48" "--config $c"
done
one "c5 default" "XC_X=0" "--config c5"
one "c5 PF=1" "XC_SPMM_PF=1" "--config c5"
one "c5 items48" "XC_WIN_ITEMS_A=48" "--config c5"
