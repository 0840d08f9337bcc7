set -o pipefail
mkdir -p gpurun_out/r6
run() { # name env config steps
  env $2 timeout 900 python bench.py --config $3 --steps $4 --warmup 2 --no-cpu-baseline > gpurun_out/r6/$1.json 2>gpurun_out/r6/$1.err
  echo "$1 $(python -c "import json;d=json.loads(open('gpurun_out/r6/$1.json').read().splitlines()[-1]);print(round(d['value'],4), round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
}
run north_qt64 "QT_QTHETA_MAX_ROWS=1000000 QT_QR_OB=64" north 5
run north_qt192 "QT_QTHETA_MAX_ROWS=1000000 QT_QR_OB=192" north 5
run c3_base "QT_QTHETA_MAX_ROWS=2048" c3 2
run c3_qt "QT_QTHETA_MAX_ROWS=1000000" c3 2
run c4_base "QT_QTHETA_MAX_ROWS=2048" c4 1
run c4_qt "QT_QTHETA_MAX_ROWS=1000000" c4 1
run c4_ob0 "QT_QR_OB=0 QT_QTHETA_MAX_ROWS=2048" c4 1
run c5_base "QT_QTHETA_MAX_ROWS=2048" c5 2
run c5_qt "QT_QTHETA_MAX_ROWS=1000000" c5 2
run c5_ob0 "QT_QR_OB=0 QT_QTHETA_MAX_ROWS=2048" c5 2
run c2 "X=1" c2 20
