set -o pipefail
mkdir -p gpurun_out/p8
python tools/profile_update.py --config north > gpurun_out/p8/pu.log 2>&1; cat gpurun_out/p8/pu.log
N0=$(grep -o "launches_before=[0-9]*" gpurun_out/p8/pu.log | cut -d= -f2); NP=$(grep -o "launches_profiled=[0-9]*" gpurun_out/p8/pu.log | cut -d= -f2)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $N0 -c $NP --csv --log-file gpurun_out/p8/launches_update_north.csv python tools/profile_update.py --config north > gpurun_out/p8/ncu1.log 2>&1; echo "ncu1 rc=$?"
python tools/launch_summary.py gpurun_out/p8/launches_update_north.csv | head -24
python tools/profile_step.py --config north > gpurun_out/p8/ps.log 2>&1; S0=$(grep -o "launches_before=[0-9]*" gpurun_out/p8/ps.log | cut -d= -f2); SP=$(grep -o "launches_profiled=[0-9]*" gpurun_out/p8/ps.log | cut -d= -f2)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $S0 -c $SP --csv --log-file gpurun_out/p8/launches_step_north.csv python tools/profile_step.py --config north > gpurun_out/p8/ncu2.log 2>&1; echo "ncu2 rc=$?"
python tools/launch_summary.py gpurun_out/p8/launches_step_north.csv | head -24
