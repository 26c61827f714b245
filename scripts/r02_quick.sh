mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_march.py -q -p no:cacheprovider > gpurun_out/t_march.log 2>&1; echo exit=$? >> gpurun_out/t_march.log
timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --nrhs 0 --no-extra > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1200 python scripts/config4_partitioned.py --ranks 4 --out gpurun_out/r02_config4_partitioned.json > gpurun_out/c4p.log 2>&1
