#!/bin/bash
# launch list (serialized kernel durations) of one eager C2 update
P=gpurun_out/prof
mkdir -p $P
python tools/profile_update.py --config c2 > $P/pu.log 2>&1 && \
N0=$(grep -o "launches_before=[0-9]*" $P/pu.log | cut -d= -f2) && \
NP=$(grep -o "launches_profiled=[0-9]*" $P/pu.log | cut -d= -f2) && \
ncu --metrics gpu__time_duration.sum --clock-control none -s $N0 -c $NP --csv --log-file $P/launches_update_c2.csv \
    python tools/profile_update.py --config c2 > $P/ncu_pu.log 2>&1
echo rc=$?
python tools/launch_summary.py $P/launches_update_c2.csv > $P/launches_update_c2_summary.txt 2>&1; head -40 $P/launches_update_c2_summary.txt
