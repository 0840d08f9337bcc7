# A/B of the split X GEMM (QT_NO_X_SPLIT=1: X in one GEMM): bench value, e2e, median step ms
for rep in 1 2 3; do
  for v in ${VARIANTS:-split nosplit}; do
    unset QT_NO_X_SPLIT
    case $v in nosplit) export QT_NO_X_SPLIT=1;; esac
    out=$(timeout 300 python bench.py --config ${CFG:-c2} --steps ${STEPS:-60} --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); import statistics as s; print(round(d['value'],2), round(d['e2e']['value'],2), 'median_ms', s.median(d['step_ms']))")
    echo "$rep ${CFG:-c2} $v $out"
  done
done
