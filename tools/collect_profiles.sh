#!/bin/bash
# ncu evidence for profiles/: launch lists of the bench commands and one
# full-set capture of the dominant DMMA GEMM (run after the plain commands exit 0)
set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_c2.log 2>&1
python tools/gemm_one.py 5120 1024 5120 --opb 1 --beta 0 > gpurun_out/plain_gemm.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:zgemm_kernel -s 1 -c 1 \
    -o gpurun_out/zgemm_x_north python tools/gemm_one.py 5120 1024 5120 --opb 1 --beta 0 > gpurun_out/ncu_gemm.log 2>&1
python tools/gemm_one.py 1024 25600 1024 --beta 0 > gpurun_out/plain_gemm2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:zgemm_kernel -s 1 -c 1 \
    -o gpurun_out/zgemm_theta_north python tools/gemm_one.py 1024 25600 1024 --beta 0 > gpurun_out/ncu_gemm2.log 2>&1
tail -2 gpurun_out/ncu_bench_c2.log gpurun_out/ncu_gemm.log gpurun_out/ncu_gemm2.log
