#!/bin/bash
# ncu launch lists (gpu__time_duration.sum, --clock-control none) of one
# default bench run and of exactly one C2 Trotter step, each after the same
# command exited 0 without ncu; then the one-GPU bench sweep
P=gpurun_out/prof
mkdir -p $P
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $P/plain_c2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_bench_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $P/ncu_bench_c2.log 2>&1
python tools/profile_step.py --config c2 > $P/ps.log 2>&1 && \
N0=$(grep -o "launches_before=[0-9]*" $P/ps.log | cut -d= -f2) && \
NP=$(grep -o "launches_profiled=[0-9]*" $P/ps.log | cut -d= -f2) && \
ncu --metrics gpu__time_duration.sum --clock-control none -s $N0 -c $NP --csv --log-file $P/launches_step_c2.csv \
    python tools/profile_step.py --config c2 > $P/ncu_step.log 2>&1
echo "launch lists rc=$?"
bash tools/bench_all.sh
