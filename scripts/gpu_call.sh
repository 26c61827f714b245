set -x
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider -x > gpurun_out/gpu_multirank.log 2>&1; echo exit=$? >> gpurun_out/gpu_multirank.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
