#!/bin/bash
# SpMM diagnostic variants (XC_SPMM_EXP: results invalid, timing only) + batch sensitivity.
mkdir -p gpurun_out
one() {  # label, env, bench args
  env $2 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline $3 > gpurun_out/exp.json 2> gpurun_out/exp.err || { echo "$1 FAILED"; tail -3 gpurun_out/exp.err; return; }
  python -c "
import json;d=json.load(open('gpurun_out/exp.json'));r=d['roofline'];print('%-14s'%'$1','B=%d'%d['config'].get('B_per_gpu',0),'ms %.3f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac']))"
}
one base "XC_X=0" "--config c5"
one nostage "XC_SPMM_EXP=1" "--config c5"
one nostore "XC_SPMM_EXP=2" "--config c5"
one twice "XC_SPMM_EXP=3" "--config c5"
one b1024 "XC_X=0" "--config c5 --batch 1024"
one b256 "XC_X=0" "--config c5 --batch 256"
one c4 "XC_X=0" "--config c4"
one c4twice "XC_SPMM_EXP=3" "--config c4"
one c3 "XC_X=0" "--config c3"
one c3twice "XC_SPMM_EXP=3" "--config c3"
