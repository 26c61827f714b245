set -x
timeout 1500 python scripts/deep_probe3.py > gpurun_out/deep3.log 2>&1; echo exit=$? >> gpurun_out/deep3.log
