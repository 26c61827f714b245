mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_march.py -q -p no:cacheprovider > gpurun_out/t_quick.log 2>&1; echo exit=$? >> gpurun_out/t_quick.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nrhs 0 --no-extra > gpurun_out/bench.json 2> gpurun_out/bench.err
HMG_NO_RRFUSE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nrhs 0 --no-extra > gpurun_out/bench_norr.json 2> gpurun_out/bench_norr.err
HMG_SMARCH=8 timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --nrhs 0 --no-extra > gpurun_out/bench_sm8.json 2> gpurun_out/bench_sm8.err
HMG_SMARCH=16 timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --nrhs 0 --no-extra > gpurun_out/bench_sm16.json 2> gpurun_out/bench_sm16.err
