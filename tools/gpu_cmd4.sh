set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest -q --timeout 600 tests/test_cbe_gpu.py tests/test_linalg_gpu.py "tests/test_headline_gpu.py::test_c3_cbe_update_parity" "tests/test_headline_gpu.py::test_c4_single_bond_matches_fixture" > gpurun_out/gt4.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^E " gpurun_out/gt4.log | head -20
QT_UPDATE_DEBUG=1 D=5 CHI=1024 timeout 300 python tools/update_probe.py > gpurun_out/upd_north.log 2>&1; tail -4 gpurun_out/upd_north.log
python tools/profile_step.py --config north > gpurun_out/ps_north.log 2>&1; cat gpurun_out/ps_north.log
N0=$(grep -o "launches_before=[0-9]*" gpurun_out/ps_north.log | cut -d= -f2); NP=$(grep -o "launches_profiled=[0-9]*" gpurun_out/ps_north.log | cut -d= -f2)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $N0 -c $NP --csv --log-file gpurun_out/launches_north.csv python tools/profile_step.py --config north > gpurun_out/ncu_north.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_north.csv | head -30
