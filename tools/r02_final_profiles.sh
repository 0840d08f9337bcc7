#!/bin/bash
# Round-2 final ncu evidence (3M GEMM build): launch lists of one north-star
# update and one step, and --set full captures of the dominant kernels at the
# north-star shapes (each command first exits 0 without ncu).
set -o pipefail
P=gpurun_out/r02f3
mkdir -p $P
python tools/profile_update.py --config north > $P/pu.log 2>&1 && \
N0=$(grep -o "launches_before=[0-9]*" $P/pu.log | cut -d= -f2) && NP=$(grep -o "launches_profiled=[0-9]*" $P/pu.log | cut -d= -f2) && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $N0 -c $NP --csv --log-file $P/launches_update_north.csv \
  python tools/profile_update.py --config north > $P/ncu_pu.log 2>&1; echo "update list rc=$?"
python tools/launch_summary.py $P/launches_update_north.csv > $P/launches_update_north_summary.txt 2>&1
python tools/profile_step.py --config north > $P/ps.log 2>&1 && \
S0=$(grep -o "launches_before=[0-9]*" $P/ps.log | cut -d= -f2) && SP=$(grep -o "launches_profiled=[0-9]*" $P/ps.log | cut -d= -f2) && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $S0 -c $SP --csv --log-file $P/launches_step_north.csv \
  python tools/profile_step.py --config north > $P/ncu_ps.log 2>&1; echo "step list rc=$?"
python tools/launch_summary.py $P/launches_step_north.csv > $P/launches_step_north_summary.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
full() {  # name kernel-regex skip command...
  local name=$1 kre=$2 skip=$3; shift 3
  "$@" > $P/plain_$name.log 2>&1 && timeout 900 $NCU -k "regex:$kre" -s $skip -c 1 -o $P/$name "$@" > $P/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
full gemm_x zgemm_kernel 1 python tools/gemm_one.py 5120 1024 5120 --opb 1 --beta 0 --reps 2
full gemm_theta zgemm_kernel 1 python tools/gemm_one.py 1024 25600 1024 --beta 0 --reps 2
full gemm_apply_w zgemm_kernel 1 python tools/gemm_one.py 128 5120 5120 --opa 1 --beta 0 --reps 2
full gemm_apply_c zgemm_kernel 1 python tools/gemm_one.py 5120 5120 128 --beta 1 --reps 2
full panel_5120 panel_cluster 1 python tools/qr_one.py 5120 64 2
full jacobi_356 jacobi_kernel 1 python tools/eigh_one.py 356
full jacobi_1127 jacobi_kernel 1 python tools/eigh_one.py 1127
python tools/ncu_summary.py $P/*.ncu-rep > $P/ncu_north_summary.txt 2>&1; cat $P/ncu_north_summary.txt
for f in $P/*.ncu-rep; do ncu -i $f --page raw --csv | gzip > ${f%.ncu-rep}_raw.csv.gz; done
rm -f $P/*.ncu-rep
du -sh $P
