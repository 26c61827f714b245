# Packed FFMA2 complex FMAs (common.cuh): full GPU suite, then config 3 / config 1 timings and the
# config-3 per-kernel breakdown.   bash scripts/r02_ffma2.sh
mkdir -p gpurun_out
ENVS="X=1" ARGS="--config 3" bash scripts/time_sweep.sh; cp gpurun_out/time_sweep.txt gpurun_out/p_sweep_c3.txt
ENVS="X=1" ARGS="--config 1 --n 4096" bash scripts/time_sweep.sh; cp gpurun_out/time_sweep.txt gpurun_out/p_sweep_c1.txt
python scripts/profile_config.py --config 3 > gpurun_out/p_config3_breakdown.txt 2>&1
cat gpurun_out/p_sweep_c3.txt gpurun_out/p_sweep_c1.txt; head -14 gpurun_out/p_config3_breakdown.txt
python -m pytest tests -m gpu -x -q > gpurun_out/p_tests.log 2>&1
echo tests_exit=$? >> gpurun_out/p_tests.log
tail -3 gpurun_out/p_tests.log
