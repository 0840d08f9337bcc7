#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box from the repo root; every
# capture runs only after the same command exited 0 without ncu):
#   * launch list (gpu__time_duration.sum, --clock-control none) of one
#     default bench invocation and of one profiled C2 Trotter step;
#   * one --set full capture of the dominant kernels: the DMMA GEMM on the C2
#     and north-star shapes, the cluster QR panel, the block reflector and the
#     Jacobi eigensolver.
set -x
mkdir -p gpurun_out/prof
P=gpurun_out/prof
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
  ncu --set full --import-source on --clock-control none -k "regex:$kre" -s $skip -c 1 -o $P/$name "$@" \
      > $P/ncu_$name.log 2>&1
}
full zgemm_c2 zgemm_kernel 1 python tools/gemm_one.py 1280 256 1280 --opb 1 --beta 0
full zgemm_north zgemm_kernel 1 python tools/gemm_one.py 5120 1024 5120 --opb 1 --beta 0
full panel_c2 panel_cluster 8 python tools/qr_one.py 1280 256 2
full larfb_c2 larfb_cluster 7 python tools/qr_one.py 1280 256 2
full jacobi_c2cbe jacobi_kernel 1 python tools/eigh_one.py 356
full larfb32_c2 larfb_cluster 0 python tools/qr_one.py 1280 256 2  # first launch: trailing update, cw = 32
full permute_c2 permute_kernel 2 python tools/profile_step.py --config c2
full transpose_c2 transpose_tiled_kernel 1 python tools/profile_step.py --config c2
# pipelined QR pair (C2 step): multi-reflector block update, Y^H extraction, Q^H theta residual
full larfbmulti_c2 larfb_multi_kernel 6 python tools/profile_step.py --config c2
full yhgauge_c2 yh_gauge_kernel 3 python tools/profile_step.py --config c2
full qtresid_c2 qtheta_resid_partial_kernel 1 python tools/profile_step.py --config c2
tail -1 $P/ncu_*.log
