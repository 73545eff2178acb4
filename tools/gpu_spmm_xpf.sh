#!/bin/bash
# X-window L2 prefetch distance sweep (XC_SPMM_XPF = CTAs ahead in grid order)
mkdir -p gpurun_out
one() {
  env $2 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline $3 > gpurun_out/exp.json 2> gpurun_out/exp.err || { echo "$1 FAILED"; tail -3 gpurun_out/exp.err; return; }
  python -c "
import json;d=json.load(open('gpurun_out/exp.json'));r=d['roofline'];print('%-14s'%'$1','B=%d'%d['config'].get('B_per_gpu',0),'ms %.3f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac']))"
}
for rep in 1 2; do
for a in 0 148 296 592; do one "c5 xpf=$a" "XC_SPMM_XPF=$a" "--config c5"; done
done
for a in 0 296; do one "c3 xpf=$a" "XC_SPMM_XPF=$a" "--config c3"; one "c4 xpf=$a" "XC_SPMM_XPF=$a" "--config c4"; done
