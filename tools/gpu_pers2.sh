#!/bin/bash
# persistent SpMM A/B (bench only) + the output-axis parity tests
mkdir -p gpurun_out
one() {
  env $2 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline $3 > gpurun_out/exp.json 2> gpurun_out/exp.err || { echo "$1 FAILED"; tail -3 gpurun_out/exp.err; return; }
  python -c "
import json;d=json.load(open('gpurun_out/exp.json'));r=d['roofline'];print('%-14s'%'$1','ms %.4f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac']))"
}
for c in c5 c3 c4; do
  for v in 0 1; do one "$c pers=$v" "XC_SPMM_PERS=$v" "--config $c"; done
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "output_axis or c5_same or c5_gpu or same_operator or determinism or graph_replay or input_axis_parity_laguerre" > gpurun_out/pytest_pers.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pers.log
