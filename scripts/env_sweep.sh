mkdir -p gpurun_out
: > gpurun_out/env3.txt
timeout 900 python -m pytest tests/test_gpu_dict.py tests/test_gpu_tail.py -q -p no:cacheprovider -x > gpurun_out/t_dict.log 2>&1; echo exit=$? >> gpurun_out/t_dict.log
for e in ${ENVS:-"X=1" "HMG_TAIL_NODES=40000" "HMG_TAIL_NODES=0"}; do
  echo "== $e" >> gpurun_out/env3.txt
  env $e timeout 300 python scripts/profile_config.py --config ${CFG:-3} 2>&1 | head -${NL:-8} >> gpurun_out/env3.txt
done
