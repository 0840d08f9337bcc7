set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest -q --timeout 600 tests/test_linalg_gpu.py tests/test_cbe_gpu.py "tests/test_headline_gpu.py::test_north_star_update_parity" > gpurun_out/gt5.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^E " gpurun_out/gt5.log | head -20
for ob in 0 128 256; do QT_QR_OB=$ob timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bn_ob$ob.json 2>gpurun_out/bn_ob$ob.err; echo "ob=$ob $(python -c "import json;d=json.loads(open('gpurun_out/bn_ob$ob.json').read().splitlines()[-1]);print(d['value'], d['roofline']['frac'])")"; done
for ob in 128 256; do QT_QTHETA_MAX_ROWS=8192 QT_QR_OB=$ob timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bn_qt$ob.json 2>gpurun_out/bn_qt$ob.err; echo "qtheta ob=$ob $(python -c "import json;d=json.loads(open('gpurun_out/bn_qt$ob.json').read().splitlines()[-1]);print(d['value'], d['roofline']['frac'])")"; done
QT_UPDATE_DEBUG=1 D=5 CHI=1024 timeout 300 python tools/update_probe.py 2>&1 | tail -2
QT_QTHETA_MAX_ROWS=8192 QT_UPDATE_DEBUG=1 D=5 CHI=1024 timeout 300 python tools/update_probe.py 2>&1 | tail -2
