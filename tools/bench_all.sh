#!/bin/bash
# every bench configuration once on one GPU (JSON lines under gpurun_out/bench_all/)
mkdir -p gpurun_out/bench_all
run() {  # name timeout args...
  local name=$1 to=$2; shift 2
  timeout $to python bench.py "$@" > gpurun_out/bench_all/$name.json 2> gpurun_out/bench_all/$name.err
  echo "$name rc=$? $(tail -1 gpurun_out/bench_all/$name.json | cut -c1-160)"
}
run default 900
run c2 400 --config c2 --steps 20 --warmup 5 --no-cpu-baseline
run c1 300 --config c1 --steps 50 --warmup 5 --no-cpu-baseline
run c2cbe 300 --config c2cbe --steps 10 --warmup 3 --no-cpu-baseline
run northcbe 400 --config northcbe --steps 4 --warmup 3 --no-cpu-baseline
run c3 600 --config c3 --steps 3 --warmup 3 --no-cpu-baseline
run c5small 300 --config c5small --steps 5 --warmup 3 --no-cpu-baseline
run c5 900 --config c5 --steps 2 --warmup 3 --no-cpu-baseline
run c4 900 --config c4 --steps 2 --warmup 3 --no-cpu-baseline
run ref_default 900 --impl reference
