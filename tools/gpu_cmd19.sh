#!/bin/bash
# Jacobi absolute-floor sweep on the CBE configs (sweeps per solve, steps/s)
set -x
QT_EIGH_DEBUG=1 timeout 120 python bench.py --config c2cbe --steps 3 --warmup 3 2>&1 | grep -E "eigh n" | tail -4
for a in 1e-22 1e-19 1e-18 1e-17; do
  QT_JACOBI_ABS=$a timeout 120 python bench.py --config c2cbe --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2cbe abs=$a', d['value'])"
  QT_EIGH_DEBUG=1 QT_JACOBI_ABS=$a timeout 120 python bench.py --config c2cbe --steps 2 --warmup 3 2>&1 | grep -E "eigh n" | tail -2
done
for a in 1e-22 1e-18; do
  QT_JACOBI_ABS=$a timeout 300 python bench.py --config c3 --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3 abs=$a', d['value'])"
  QT_EIGH_DEBUG=1 QT_JACOBI_ABS=$a timeout 300 python bench.py --config c3 --steps 1 --warmup 3 2>&1 | grep -E "eigh n" | tail -2
done
