#!/bin/bash
# one-pass C2R (c2r1.cu): engine + parity tests, then A/B against the two-pass form (XC_C2R_ONE=0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "c2r_engine or output_axis or c5_same or c5_gpu or same_operator or determinism or lag2d_parity" > gpurun_out/pytest_one.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_one.log
one() {
  env $2 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline $3 > gpurun_out/exp.json 2> gpurun_out/exp.err || { echo "$1 FAILED"; tail -3 gpurun_out/exp.err; return; }
  python -c "
import json;d=json.load(open('gpurun_out/exp.json'));r=d['roofline'];print('%-14s'%'$1','ms %.4f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac']))"
}
for c in c5 c3 c4 c8 c5n32k; do
  for v in 0 1; do one "$c one=$v" "XC_C2R_ONE=$v" "--config $c"; done
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "xc_apply/" --csv --log-file gpurun_out/launches_one.csv python bench.py --config c5 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches_one.csv 9 > gpurun_out/launches_one.txt; head -14 gpurun_out/launches_one.txt
