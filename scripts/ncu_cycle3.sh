mkdir -p gpurun_out
HMG_NO_GRAPHS=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -f -o /tmp/c3cycle python scripts/ncu_cycle.py --config 3 > gpurun_out/ncu_c3.log 2>&1
python scripts/ncu_summary.py full /tmp/c3cycle.ncu-rep gpurun_out/ncu_c3_full.md > /dev/null 2>&1
ncu -i /tmp/c3cycle.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/c3_raw.csv.gz
ls -la gpurun_out
