#!/bin/bash
# Jacobi: end-of-sweep scan + single-barrier inner rounds -- tests and timing
python -m pytest tests/test_cbe_gpu.py tests/test_linalg_gpu.py -x -q 2>&1 | tail -3
QT_EIGH_DEBUG=1 timeout 120 python bench.py --config c2cbe --steps 2 --warmup 3 2>&1 | grep -E "eigh n" | tail -2
timeout 120 python bench.py --config c2cbe --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2cbe', d['value'])"
QT_EIGH_DEBUG=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 3 2>&1 | grep -E "eigh n" | tail -2
timeout 300 python bench.py --config c3 --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3', d['value'])"
