mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage3d.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/t_quick.log 2>&1; echo exit=$? >> gpurun_out/t_quick.log
timeout 600 python scripts/profile_config.py --config 3 > gpurun_out/prof3.txt 2>&1
timeout 600 python scripts/bench_configs.py --only 3 --out gpurun_out/cfg3.jsonl > gpurun_out/cfg3.log 2>&1
