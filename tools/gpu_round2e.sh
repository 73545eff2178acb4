#!/bin/bash
# Round-2 GPU evidence in one call: the GPU test suite, every bench line (with the CPU oracle leg),
# the reference arm, the c5 parity record, the c5 launch list and an ncu --set full of the c5 SpMM.
mkdir -p gpurun_out/r02e
O=gpurun_out/r02e
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 rc=$?"; cat $O/bench_c5.json
for c in c1 c2 c3 c4 c6 c7 c8 c5n32k c5n128k; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --e2e-steps 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
timeout 300 python bench.py --config c4 --direction WAT --steps 10 --warmup 3 --e2e-steps 3 > $O/bench_c4_wat.json 2> $O/bench_c4_wat.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference_c5.json 2>&1; echo "ref rc=$?"
timeout 600 python tools/c5_parity_record.py > $O/c5_parity.json 2>&1
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "xc_apply/" --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
CMD2="python bench.py --config c5 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD2 > $O/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_win -s 2 -c 1 -o $O/prof_spmm_c5 $CMD2 > $O/ncu_spmm.log 2>&1; echo "ncu spmm rc=$?"

python tools/c1_host_probe.py c1 > $O/c1_host_probe.txt 2>&1
CMD3="python bench.py --config c3 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD3 > $O/plain3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "xc_apply/" --csv --log-file $O/launches_c3.csv $CMD3 > $O/ncu_launches_c3.log 2>&1; echo "ncu c3 rc=$?"
echo all-done
