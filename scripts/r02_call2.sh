set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_uniform.py tests/test_gpu_golden.py -q -p no:cacheprovider -x > gpurun_out/t_uniform.log 2>&1; echo exit=$? >> gpurun_out/t_uniform.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nrhs 0 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$? >> gpurun_out/bench.err
HMG_NO_UNIFORM=1 timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --nrhs 0 > gpurun_out/bench_nouni.json 2> gpurun_out/bench_nouni.err
