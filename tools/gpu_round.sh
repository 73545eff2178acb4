#!/bin/bash
# One GPU call: GPU tests, the default bench line, per-config bench lines, then the
# profiles (launch list + ncu --set full of the SpMM and FFT passes).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc=$?"
cat gpurun_out/bench_c5.json
for c in c1 c2 c3 c4 c6 c7 c8; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python bench.py --config c4 --direction WAT --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c4_wat.json 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
[ "$1" = "noprof" ] || timeout 1200 bash tools/gpu_profile_round.sh
echo done
