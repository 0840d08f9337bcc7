#!/bin/bash
# theta-side (side2) stream priority A/B on C2, C2-CBE and the north star
python -c "import torch; print(torch.cuda.Stream.priority_range())"
for p in 0 1 2; do
  for c in c2 c2cbe; do
    QT_SIDE2_PRIO=$p timeout 120 python bench.py --config $c --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('prio $p $c', round(d['value'],2))"
  done
  QT_SIDE2_PRIO=$p timeout 300 python bench.py --config north --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('prio $p north', round(d['value'],3))"
done
