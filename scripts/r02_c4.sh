mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_streams.py tests/test_gpu_damping.py -q -p no:cacheprovider > gpurun_out/t_streams.log 2>&1; echo exit=$? >> gpurun_out/t_streams.log
timeout 2400 python scripts/config4_sweep.py --out gpurun_out/r02_config4_sweep.jsonl > gpurun_out/c4.log 2>&1
