set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$? >> gpurun_out/bench.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 60000 -c 3000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo ncu_list_exit=$? >> gpurun_out/ncu_list.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_smooth_stored2d|k_rb2d_march|k_multi_axpy|k_multidot|k_stored_op|k_prolong" -s 400 -c 12 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full_exit=$? >> gpurun_out/ncu_full.log
