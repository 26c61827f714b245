# Round-2 evidence on one B200 (run through gpurun from the repo root).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo exit=$? >> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo exit=$? >> gpurun_out/ref.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --nrhs 0 --no-extra"
if timeout 600 $CMD > gpurun_out/bench_s1.json 2> gpurun_out/bench_s1.err; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 60000 -c 3000 --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
  timeout 1200 ncu -f --set full --clock-control none --import-source on \
      -k regex:"k_multi_axpy_f4|k_multidot_f4" -s 400 -c 40 -o /tmp/kry $CMD > gpurun_out/ncu_kry.log 2>&1
  timeout 1200 ncu -f --set full --clock-control none --import-source on \
      -k regex:"k_stored_op2d_pair|k_rb2d_march2|k_vanka_stencil|k_prolong_block|k_restrict_pair|k_fine_op2d_march" \
      -s 2000 -c 24 -o /tmp/full $CMD > gpurun_out/ncu_full.log 2>&1
  python scripts/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/r02_launches_bench_n4096_c64.md
  python scripts/ncu_summary.py full /tmp/kry.ncu-rep gpurun_out/r02_ncu_krylov_n4096_c64.md --traffic-key "multi_axpy@L0|c64|4096" --traffic-kernel k_multi_axpy
  python scripts/ncu_summary.py full /tmp/full.ncu-rep gpurun_out/r02_ncu_full_bench_n4096_c64.md
  cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json 2>/dev/null
  ncu -i /tmp/full.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/full_raw.csv.gz
  ncu -i /tmp/kry.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/kry_raw.csv.gz
fi
timeout 900 python scripts/bench_configs.py --out gpurun_out/r02_configs.jsonl > gpurun_out/configs.log 2>&1
ls -la gpurun_out
