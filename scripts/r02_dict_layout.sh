# Plane-major dictionary tables (k_dict.cuh): dictionary / tail tests, then config 3 and config 1 timings
# and the config-3 per-kernel breakdown.   bash scripts/r02_dict_layout.sh
mkdir -p gpurun_out
python -m pytest tests/test_gpu_dict.py tests/test_gpu_tail.py -x -q > gpurun_out/d_tests.log 2>&1
echo tests_exit=$? >> gpurun_out/d_tests.log
tail -3 gpurun_out/d_tests.log
ENVS="X=1 HMG_NO_DICT=1" ARGS="--config 3" bash scripts/time_sweep.sh; cp gpurun_out/time_sweep.txt gpurun_out/d_sweep_c3.txt
ENVS="X=1" ARGS="--config 1 --n 4096" bash scripts/time_sweep.sh; cp gpurun_out/time_sweep.txt gpurun_out/d_sweep_c1.txt
python scripts/profile_config.py --config 3 > gpurun_out/d_config3_breakdown.txt 2>&1
cat gpurun_out/d_sweep_c3.txt gpurun_out/d_sweep_c1.txt; head -24 gpurun_out/d_config3_breakdown.txt
