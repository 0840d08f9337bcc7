#!/bin/bash
# Jacobi block width A/B at n=356 (C2-CBE) and n=1127 (C3)
for jb in 16 32; do
  QT_JACOBI_JB=$jb QT_EIGH_DEBUG=1 timeout 120 python bench.py --config c2cbe --steps 2 --warmup 2 2>&1 | grep -E "eigh n" | tail -1
  QT_JACOBI_JB=$jb QT_EIGH_DEBUG=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 1 2>&1 | grep -E "eigh n" | tail -1
done
