set -x
python scripts/vcycle_probe.py > gpurun_out/probe.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:galerkin1_mf -c 1 -o gpurun_out/mf1 python scripts/vcycle_probe.py > gpurun_out/ncu_mf.log 2>&1
