#!/bin/bash
# make_rot formula A/B (old 4-deep chain vs 2-deep), Jacobi timings at n=356 / 1127
cd paper_2212_09782_b200
for v in new old; do
  if [ $v = old ]; then touch csrc/jacobi.cu; make XFLAGS=-DQT_JACOBI_OLD_ROT >/dev/null 2>&1 || exit 1; fi
  cd ..
  echo "== $v"
  QT_EIGH_DEBUG=1 timeout 120 python bench.py --config c2cbe --steps 2 --warmup 3 2>&1 | grep -E "eigh n" | tail -1
  QT_EIGH_DEBUG=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 2 2>&1 | grep -E "eigh n" | tail -1
  cd paper_2212_09782_b200
done
touch csrc/jacobi.cu; make >/dev/null 2>&1
