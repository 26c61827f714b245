# Round evidence on one B200 (run through gpurun from the repo root).
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo exit=$? >> gpurun_out/bench_full.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --nrhs 0"
if timeout 600 $CMD > gpurun_out/bench_s1.json 2> gpurun_out/bench_s1.err; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 60000 -c 3000 --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on \
      -k regex:"k_stored_op|k_rb2d_march|k_vanka_stencil|k_multi_axpy|k_multidot|k_prolong_block|k_restrict|k_fine_op" \
      -c 40 -o /tmp/full $CMD > gpurun_out/ncu_full.log 2>&1
  python scripts/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/launches.md
  python scripts/ncu_summary.py full /tmp/full.ncu-rep gpurun_out/full.md --traffic-key "stored_residual@L1|c64|4096" --traffic-kernel k_stored_op
  ncu -i /tmp/full.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/full_raw.csv.gz
  ls -la gpurun_out
fi
timeout 1500 python scripts/bench_configs.py --out gpurun_out/configs.jsonl > gpurun_out/configs.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo exit=$? >> gpurun_out/ref.err
