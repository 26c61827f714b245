set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not config4_s4" > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nrhs 0 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$? >> gpurun_out/bench.err
