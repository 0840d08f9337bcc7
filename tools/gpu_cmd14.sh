set -o pipefail
timeout 900 python -m pytest -q --timeout 600 tests/test_headline_gpu.py tests/test_qr_pair_gpu.py -x > gpurun_out/gt14.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^E " gpurun_out/gt14.log | head -20
for v in 1 0; do QT_NO_TALL_PAIR=$( [ $v = 1 ] && echo 1 ) timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-scaling-anchor > gpurun_out/b14_$v.json 2>&1; echo "notall=$v $(python -c "import json;d=json.loads(open('gpurun_out/b14_$v.json').read().splitlines()[-1]);print(d['value'], d['roofline']['frac'])" 2>&1 | tail -1)"; done
QT_UPDATE_DEBUG=1 D=5 CHI=1024 timeout 300 python tools/update_probe.py 2>&1 | tail -1
