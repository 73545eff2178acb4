#!/bin/bash
# One GPU call: bench (all configs), then ncu launch list + full capture of the SpMM.
set -x
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?"
for c in c1 c2 c3 c4; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --config c4 --direction WAT --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c4_wat.json 2>&1
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"spmm|fft_pass|reduce_rows" --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_dmma -s 3 -c 1 -o gpurun_out/prof_spmm -f $CMD > gpurun_out/ncu_full.log 2>&1
echo done
