# Source-level ncu captures of selected kernels on the bench workload (V-cycle probe).
set -x
python scripts/vcycle_probe.py > gpurun_out/probe.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_rb2d_march2" -c 2 -o /tmp/sel python scripts/vcycle_probe.py > gpurun_out/ncu_sel.log 2>&1
for i in 0 1; do
  ncu -i /tmp/sel.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 2>/dev/null | gzip > gpurun_out/sel_src_$i.csv.gz
done
ncu -i /tmp/sel.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/sel_raw.csv.gz
