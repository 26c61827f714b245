mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py tests/test_gpu_batch.py -q -p no:cacheprovider > gpurun_out/t_multi.log 2>&1; echo exit=$? >> gpurun_out/t_multi.log
