for cfg in c2 north; do for impl in reference port; do
QT_REF_IMPL=$impl timeout 600 python bench.py --impl reference --config $cfg --steps 10 --warmup 3 > gpurun_out/ref12_${cfg}_$impl.json 2>&1
echo "$cfg $impl $(python -c "import json;d=json.loads(open('gpurun_out/ref12_${cfg}_$impl.json').read().splitlines()[-1]);print(d['value'], d['cpu_baseline']['kind'], d['cpu_baseline']['sample'][:60])")"
done; done
