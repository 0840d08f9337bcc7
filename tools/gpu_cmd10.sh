set -o pipefail
mkdir -p gpurun_out/ncu10
NCU="ncu --set full --clock-control none --import-source on"
P="python tools/profile_update.py --config north"
timeout 900 $NCU -k regex:zgemm_kernel -s 388 -c 4 -o gpurun_out/ncu10/north_theta_x $P > gpurun_out/ncu10/a.log 2>&1; echo "a rc=$?"
timeout 900 $NCU -k regex:zgemm_kernel -s 408 -c 3 -o gpurun_out/ncu10/north_thetaapply $P > gpurun_out/ncu10/b.log 2>&1; echo "b rc=$?"
timeout 900 $NCU -k regex:zgemm_kernel -s 775 -c 1 -o gpurun_out/ncu10/north_hastings $P > gpurun_out/ncu10/c.log 2>&1; echo "c rc=$?"
timeout 900 $NCU -k regex:panel_cluster -s 80 -c 1 -o gpurun_out/ncu10/north_panel $P > gpurun_out/ncu10/d.log 2>&1; echo "d rc=$?"
ls -la gpurun_out/ncu10
python tools/ncu_summary.py gpurun_out/ncu10/*.ncu-rep > gpurun_out/ncu10/summary.txt 2>&1; cat gpurun_out/ncu10/summary.txt
for f in gpurun_out/ncu10/*.ncu-rep; do ncu -i $f --page raw --csv | gzip > ${f%.ncu-rep}_raw.csv.gz; done
rm -f gpurun_out/ncu10/north_theta_x.ncu-rep gpurun_out/ncu10/north_thetaapply.ncu-rep gpurun_out/ncu10/north_hastings.ncu-rep
du -sh gpurun_out
