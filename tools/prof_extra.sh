set -x
mkdir -p gpurun_out/prof
P=gpurun_out/prof
full() {  # name kernel-regex skip command...
  local name=$1 kre=$2 skip=$3; shift 3
  "$@" > $P/plain_$name.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k "regex:$kre" -s $skip -c 1 -o $P/$name "$@" \
      > $P/ncu_$name.log 2>&1
}
full larfb32_c2 larfb_cluster 0 python tools/qr_one.py 1280 256 2  # first launch: trailing update, cw = 32
full permute_c2 permute_kernel 2 python tools/profile_step.py --config c2
full transpose_c2 transpose_tiled_kernel 1 python tools/profile_step.py --config c2
full panel_c2 panel_cluster 8 python tools/qr_one.py 1280 256 2
ls $P
