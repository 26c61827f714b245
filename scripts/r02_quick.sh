mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_stage3d.py tests/test_gpu_uniform.py -q -p no:cacheprovider -x > gpurun_out/t_quick.log 2>&1; echo exit=$? >> gpurun_out/t_quick.log
timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --nrhs 0 --no-extra > gpurun_out/bench.json 2> gpurun_out/bench.err
