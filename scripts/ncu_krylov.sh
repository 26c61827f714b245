# ncu --set full on steady-state Krylov launches of the bench workload (after the same command ran clean)
set -x
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --nrhs 0"
if timeout 600 $CMD > gpurun_out/kr_plain.json 2> gpurun_out/kr_plain.err; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_multidot_f4|k_multi_axpy_f4" -s 300 -c 6 -o /tmp/kr $CMD > gpurun_out/ncu_kr.log 2>&1
  python scripts/ncu_summary.py full /tmp/kr.ncu-rep gpurun_out/kr.md
  ncu -i /tmp/kr.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/kr_raw.csv.gz
fi
