#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run first, then the launch list of the bench
# command, then one --set full capture of the sweep kernel.  Run under gpurun from the repo root.
#   bash tools/run_profile.sh config4 bin2_tma_kernel
set -u
WL=${1:-config4}
KREGEX=${2:-bin2q_kernel}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu-baseline"
$BENCH > $OUT/plain_bench_$WL.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$WL.csv $BENCH > $OUT/ncu_list_$WL.log 2>&1 && \
python tools/ncu_driver.py --workload $WL --sweeps 4 > $OUT/plain_driver_$WL.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 2 -c 1 \
    -o $OUT/prof_$WL -f python tools/ncu_driver.py --workload $WL --sweeps 4 \
    > $OUT/ncu_full_$WL.log 2>&1
echo "profile $WL rc=$?"
