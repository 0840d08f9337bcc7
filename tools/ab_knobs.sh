# Interleaved C2 A/B of the opt-in environment knobs against the default path
for rep in 1 2 3; do
  for v in base QT_HASTINGS_SPLIT QT_QB_HASTINGS QT_FUSED_PANEL QT_APPLY_COLS; do
    if [ $v = base ]; then envs=""; else envs="$v=1"; fi
    out=$(env $envs timeout 300 python bench.py --config ${CFG:-c2} --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); import statistics as s; print(round(d['value'],2), round(d['e2e']['value'],2), 'median_ms', s.median(d['step_ms']))")
    echo "$rep ${CFG:-c2} $v $out"
  done
done
