# Flat (x, y) thread indexing of the register-blocked 3D stencils: A/B timings, breakdown, full GPU suite.
mkdir -p gpurun_out
ENVS="X=1 HMG_NO_FLAT3D=1 X=2" ARGS="--config 3" bash scripts/time_sweep.sh; cp gpurun_out/time_sweep.txt gpurun_out/x_sweep_c3.txt
python scripts/profile_config.py --config 3 > gpurun_out/x_config3_breakdown.txt 2>&1
cat gpurun_out/x_sweep_c3.txt; head -14 gpurun_out/x_config3_breakdown.txt
python -m pytest tests -m gpu -x -q > gpurun_out/x_tests.log 2>&1
echo tests_exit=$? >> gpurun_out/x_tests.log
tail -3 gpurun_out/x_tests.log
