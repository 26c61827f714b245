set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$? >> gpurun_out/bench.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_multi_axpy|k_multidot" -s 300 -c 6 -o gpurun_out/prof_kr $CMD > gpurun_out/ncu_kr.log 2>&1; echo ncu_exit=$? >> gpurun_out/ncu_kr.log
