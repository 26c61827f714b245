# Full GPU check of the current tree: pytest -m gpu, bench line, config sweep, config-3 breakdown
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo exit=$? >> gpurun_out/bench_full.err
timeout 600 python scripts/profile_config.py --config 3 > gpurun_out/prof3.txt 2>&1
timeout 1500 python scripts/bench_configs.py --out gpurun_out/configs.jsonl > gpurun_out/configs.log 2>&1
