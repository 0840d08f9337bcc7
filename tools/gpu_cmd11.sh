for v in 0 1; do QT_HASTINGS_QN=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-scaling-anchor > gpurun_out/b11_$v.json 2>&1; echo "qn=$v $(python -c "import json;d=json.loads(open('gpurun_out/b11_$v.json').read().splitlines()[-1]);print(d['value'], d['roofline']['frac'])")"; done
QT_UPDATE_DEBUG=1 D=5 CHI=1024 timeout 300 python tools/update_probe.py 2>&1 | tail -1
timeout 600 python -m pytest -q tests/test_headline_gpu.py::test_north_star_update_parity 2>&1 | tail -1
