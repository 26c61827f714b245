# Warp-uniform dictionary branch (k_vanka_stencil*, k_stored_op): timings first, then the full GPU suite.
mkdir -p gpurun_out
ENVS="X=1" ARGS="--config 3" bash scripts/time_sweep.sh; cp gpurun_out/time_sweep.txt gpurun_out/w_sweep_c3.txt
ENVS="X=1" ARGS="--config 1 --n 4096" bash scripts/time_sweep.sh; cp gpurun_out/time_sweep.txt gpurun_out/w_sweep_c1.txt
python scripts/profile_config.py --config 3 > gpurun_out/w_config3_breakdown.txt 2>&1
cat gpurun_out/w_sweep_c3.txt gpurun_out/w_sweep_c1.txt; head -14 gpurun_out/w_config3_breakdown.txt
python -m pytest tests -m gpu -x -q > gpurun_out/w_tests.log 2>&1
echo tests_exit=$? >> gpurun_out/w_tests.log
tail -3 gpurun_out/w_tests.log
