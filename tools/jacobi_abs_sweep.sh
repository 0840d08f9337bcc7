for A in 1e-22 1e-18 1e-16 1e-14; do
  echo "== QT_JACOBI_ABS=$A"
  QT_JACOBI_ABS=$A QT_EIGH_DEBUG=1 python tools/eigh_one.py 356 2>&1 | grep eigh | tail -1
  QT_JACOBI_ABS=$A timeout 300 python -m pytest tests/test_cbe_gpu.py tests/test_tebd_gpu.py -q -x --timeout 200 2>&1 | tail -2
  QT_JACOBI_ABS=$A timeout 300 python bench.py --config c2cbe --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-200
done
