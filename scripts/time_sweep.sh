# time_solve.py under a list of switches:  ENVS="X=1 HMG_TAIL_NODES=20000" ARGS="--config 1 --n 4096" bash scripts/time_sweep.sh
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv,noheader > gpurun_out/time_sweep.txt
for e in ${ENVS:-X=1}; do
  env $e TAG=$e timeout 600 python scripts/time_solve.py ${ARGS:---config 1 --n 4096} >> gpurun_out/time_sweep.txt 2>&1
done
