#!/bin/bash
# every bench configuration once on one GPU (JSON lines under gpurun_out/bench_all/)
mkdir -p gpurun_out/bench_all
run() {  # name timeout args...
  local name=$1 to=$2; shift 2
  timeout $to python bench.py "$@" > gpurun_out/bench_all/$name.json 2> gpurun_out/bench_all/$name.err
  echo "$name rc=$? $(cut -c1-160 gpurun_out/bench_all/$name.json)"
}
run c2 400
run c1 300 --config c1 --steps 50 --warmup 5 --no-cpu-baseline
run c2cbe 300 --config c2cbe --steps 10 --warmup 3 --no-cpu-baseline
run north 400 --config north --steps 3 --warmup 3 --no-cpu-baseline
run northcbe 400 --config northcbe --steps 3 --warmup 3 --no-cpu-baseline
run c3 600 --config c3 --steps 2 --warmup 3 --no-cpu-baseline
run c5small 300 --config c5small --steps 5 --warmup 3 --no-cpu-baseline
run c5 900 --config c5 --steps 1 --warmup 3 --no-cpu-baseline
run c4 900 --config c4 --steps 1 --warmup 3 --no-cpu-baseline
run ref_c2 400 --impl reference
