mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/t_quick.log 2>&1; echo exit=$? >> gpurun_out/t_quick.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nrhs 0 --no-extra > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python scripts/profile_config.py --config 3 > gpurun_out/prof3.txt 2>&1
