# profile_config.py under a list of build/call-time switches, after the given tests
#   TESTS="tests/test_gpu_dict.py" ENVS="X=1 HMG_TAIL_MINB=2" CFG=3 NL=12 bash scripts/env_sweep.sh
mkdir -p gpurun_out
: > gpurun_out/env3.txt
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest $TESTS -q -p no:cacheprovider -x > gpurun_out/t_env.log 2>&1; echo exit=$? >> gpurun_out/t_env.log
fi
for e in ${ENVS:-X=1}; do
  echo "== $e" >> gpurun_out/env3.txt
  env $e timeout 300 python scripts/profile_config.py --config ${CFG:-3} 2>&1 | head -${NL:-8} >> gpurun_out/env3.txt
done
