# Refresh the bench line and the config sweep after a host-side change (kernels unchanged).
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo exit=$? >> gpurun_out/bench_full.err
timeout 1500 python scripts/bench_configs.py --out gpurun_out/configs.jsonl > gpurun_out/configs.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
