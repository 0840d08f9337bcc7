#!/bin/bash
# ncu evidence for the pipelined QR pair (run on the GPU box from the repo
# root): launch lists of one default bench run and of one C2 step, and
# --set full captures of the pair's new kernels; the .ncu-rep files are
# summarised (tools/ncu_summary.py) and exported as details CSVs on the box,
# then deleted so gpurun_out/ stays small.
set -x
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
full() {  # name kernel-regex skip command...
  local name=$1 kre=$2 skip=$3; shift 3
  "$@" > $P/plain_$name.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k "regex:$kre" -s $skip -c 1 -o /tmp/prof_$name "$@" \
      > $P/ncu_$name.log 2>&1 && \
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > $P/${name}_details.csv 2>/dev/null
}
full larfbmulti_c2 larfb_multi_kernel 6 python tools/profile_step.py --config c2
full yhgauge_c2 yh_gauge_kernel 3 python tools/profile_step.py --config c2
full qtresid_c2 qtheta_resid_partial_kernel 1 python tools/profile_step.py --config c2
full panel_c2 panel_cluster 8 python tools/qr_one.py 1280 256 2
python tools/ncu_summary.py /tmp/prof_*.ncu-rep > $P/ncu_full_summary.txt 2>&1
rm -f /tmp/prof_*.ncu-rep
ls -la $P
