# A/B of the split X GEMM (QT_NO_X_SPLIT=1 forms X in one GEMM): C2 bench value and e2e
for rep in 1 2 3 4 5; do
  for v in split nosplit; do
    if [ $v = nosplit ]; then export QT_NO_X_SPLIT=1; else unset QT_NO_X_SPLIT; fi
    out=$(timeout 300 python bench.py --config ${CFG:-c2} --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); import statistics as s; print(round(d['value'],2), round(d['e2e']['value'],2), 'median_ms', s.median(d['step_ms']))")
    echo "$rep ${CFG:-c2} $v $out"
  done
done
