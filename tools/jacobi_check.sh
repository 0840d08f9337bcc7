#!/bin/bash
# Jacobi change check: eigh / CBE tests, solve times at n = 356 / 1127, CBE configs
timeout 300 python -m pytest tests/test_cbe_gpu.py tests/test_linalg_gpu.py -x -q 2>&1 | tail -1
QT_EIGH_DEBUG=1 timeout 300 python bench.py --config c2cbe --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | grep -E "eigh n" | tail -1
QT_EIGH_DEBUG=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "eigh n" | tail -1
for c in c2cbe northcbe; do
  timeout 600 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$c', round(d['value'],3), round(d['roofline']['frac'],3))"
done
