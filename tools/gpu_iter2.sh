#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "small_path or output_axis or determinism" > gpurun_out/pytest_small.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_small.log
for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
  python -c "
import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c','%.0f/s'%d['value'],'us %.2f'%(1e3*d['ms_per_step']),'eager %.2f us'%(1e3*d['graph']['eager_ms_per_step']),'launches',d['gpu_launches'], 'spmm frac %.3f'%d['roofline']['frac'])"
done
VARIANTS="XC_SPMM_NOPF=1" bash tools/gpu_iter.sh
VARIANTS="XC_SPMM_NOPF=1" bash tools/gpu_iter.sh --config c3
