#!/bin/bash
# 3M vs 4M complex GEMM: accuracy, single-GEMM timing, bench configs
cd paper_2212_09782_b200
for v in 3m 4m; do
  if [ $v = 4m ]; then touch csrc/zgemm.cu; make XFLAGS=-DQT_ZGEMM_4M >/dev/null 2>&1 || exit 1; fi
  cd ..
  echo "== $v"
  python tools/gemm_check.py
  for s in "5120 1024 5120" "5120 5120 1024" "1280 1280 256" "1024 5120 5120"; do python tools/gemm_one.py $s --reps 5; done
  python tools/gemm_one.py 5120 1024 5120 --opb 1 --reps 5
  timeout 300 python bench.py --config north --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('north', round(d['value'],3), d['roofline']['frac'])"
  timeout 120 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2', round(d['value'],2))"
  cd paper_2212_09782_b200
done
touch csrc/zgemm.cu; make >/dev/null 2>&1
