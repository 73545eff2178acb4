#!/bin/bash
# Profiles for profiles/: launch list of the timed region (nvtx range xc_apply) and full
# captures of the SpMM and the first FFT passes.  Each ncu run follows a plain run of the
# same command that exited 0.
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline $*"
$CMD > gpurun_out/plain_round.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_round.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "xc_apply/" --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "xc_apply/" -k regex:"spmm_win|c2r_pass" -c 3 -o gpurun_out/prof_round -f $CMD > gpurun_out/ncu_round.log 2>&1
tail -2 gpurun_out/ncu_round.log
