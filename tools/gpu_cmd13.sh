set -o pipefail
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/gt13.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gt13.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
for cfg in north c2 c1; do timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-scaling-anchor > gpurun_out/b13_$cfg.json 2>&1; echo "$cfg $(python -c "import json;d=json.loads(open('gpurun_out/b13_$cfg.json').read().splitlines()[-1]);print(d['value'], d['roofline']['frac'], d['e2e']['value'])")"; done
