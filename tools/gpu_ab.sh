#!/bin/bash
# A/B of two builds on one box: paper_2004_11610_b200/libxc_base.so vs libxc_new.so (copied over
# libxc.so in turn), CFGS configs, ROUNDS alternations
mkdir -p gpurun_out
L=paper_2004_11610_b200
if [ -n "$PYTEST_K" ]; then
  cp $L/libxc_new.so $L/libxc.so
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$PYTEST_K" > gpurun_out/pytest_ab.log 2>&1; echo "pytest(new) rc=$?"; tail -2 gpurun_out/pytest_ab.log
fi
for r in $(seq ${ROUNDS:-2}); do
for v in base new; do
  cp $L/libxc_$v.so $L/libxc.so
  for cfg in ${CFGS:-c5 c3}; do
    timeout 300 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "
import json;d=json.load(open('gpurun_out/ab.json'));r=d['roofline'];print('$v $cfg','%.0f/s'%d['value'],'ms %.4f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac']))" || tail -2 gpurun_out/ab.err
  done
done
done
cp $L/libxc_new.so $L/libxc.so
