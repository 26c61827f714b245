# ncu --set full of one V-cycle:  CFG=1 bash scripts/ncu_cycle_cfg.sh  -> gpurun_out/ncu_c${CFG}_full.md, c${CFG}_raw.csv.gz
mkdir -p gpurun_out
C=${CFG:-1}
HMG_NO_GRAPHS=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on ${NCU_EXTRA} -f -o /tmp/cyc python scripts/ncu_cycle.py --config $C > gpurun_out/ncu_c${C}.log 2>&1
python scripts/ncu_summary.py full /tmp/cyc.ncu-rep gpurun_out/ncu_c${C}_full.md > /dev/null 2>&1
ncu -i /tmp/cyc.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/c${C}_raw.csv.gz
if [ -n "$SRC_KERNEL" ]; then
  ncu -i /tmp/cyc.ncu-rep --page source --csv -k regex:"$SRC_KERNEL" 2>/dev/null | gzip > gpurun_out/c${C}_src.csv.gz
fi
