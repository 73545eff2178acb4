#!/bin/bash
# persistent SpMM: parity suite + A/B against the windowed kernel (XC_SPMM_PERS=0)
mkdir -p gpurun_out
one() {
  env $2 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline $3 > gpurun_out/exp.json 2> gpurun_out/exp.err || { echo "$1 FAILED"; tail -3 gpurun_out/exp.err; return; }
  python -c "
import json;d=json.load(open('gpurun_out/exp.json'));r=d['roofline'];print('%-14s'%'$1','ms %.4f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac']))"
}
for c in c5 c3 c4 c2; do
  for v in 0 1; do one "$c pers=$v" "XC_SPMM_PERS=$v" "--config $c"; done
done
one "c4wat pers=0" "XC_SPMM_PERS=0" "--config c4 --direction WAT"
one "c4wat pers=1" "XC_SPMM_PERS=1" "--config c4 --direction WAT"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_pers.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pers.log
