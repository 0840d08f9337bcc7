# A/B of the X head width (QT_X_HEAD: columns formed on the main stream before the pair) on C2
for rep in 1 2 3; do
  for v in 64 96 128; do
    out=$(QT_X_HEAD=$v timeout 300 python bench.py --config ${CFG:-c2} --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); import statistics as s; print(round(d['value'],2), round(d['e2e']['value'],2), 'median_ms', s.median(d['step_ms']))")
    echo "$rep ${CFG:-c2} x_head=$v $out"
  done
done
