#!/bin/bash
# one GPU iteration: tests, launch list of one C2 step, bench lines
set -o pipefail
timeout 400 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -4
python tools/profile_step.py --config ${CFG:-c2} > gpurun_out/ps.log 2>&1 && N0=$(grep -o "launches_before=[0-9]*" gpurun_out/ps.log | cut -d= -f2) && NP=$(grep -o "launches_profiled=[0-9]*" gpurun_out/ps.log | cut -d= -f2) && ncu --metrics gpu__time_duration.sum --clock-control none -s $N0 -c $NP --csv --log-file gpurun_out/launches_${CFG:-c2}.csv python tools/profile_step.py --config ${CFG:-c2} > gpurun_out/ncu_step.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err; cut -c1-330 gpurun_out/bench_c2.json
timeout 300 python bench.py --config north --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_north.json 2>gpurun_out/bench_north.err; cut -c1-330 gpurun_out/bench_north.json
