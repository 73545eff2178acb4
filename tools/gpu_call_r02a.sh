mkdir -p gpurun_out
python tools/c5_parity_record.py > gpurun_out/c5_parity.json 2>&1; echo "parity rc=$?"; cat gpurun_out/c5_parity.json
for c in c5n32k c5n128k; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
  python -c "
import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];print('$c','%.0f/s'%d['value'],'ms %.3f'%d['ms_per_step'],'spmm %.3f fft %.3f frac %.3f step_frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac'],r['step_frac']))"
done
XC_C2R_LOG=1 timeout 600 python bench.py --config c5n128k --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 >/dev/null | grep "c2r generic" | sort | uniq -c
bash tools/gpu_sanitize.sh memcheck
