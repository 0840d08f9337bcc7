set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest -q --timeout 600 tests/test_chain_gpu.py tests/test_qr_pair_gpu.py tests/test_cpp_api.py tests/test_finite_gpu.py > gpurun_out/gt9.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^E " gpurun_out/gt9.log | head -20
timeout 600 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/b9_c5.json 2>gpurun_out/b9_c5.err; echo "c5 rc=$?"; cut -c1-300 gpurun_out/b9_c5.json; tail -3 gpurun_out/b9_c5.err
timeout 900 python bench.py > gpurun_out/b9_default.json 2>gpurun_out/b9_default.err; echo "default rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/b9_default.json').read().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['e2e'],d.get('cpu_baseline',{}).get('value'),d.get('scaling_anchor'))"
