mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nrhs 0 --no-extra > gpurun_out/bench.json 2> gpurun_out/bench.err
HMG_PDL=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nrhs 0 --no-extra > gpurun_out/bench_pdl.json 2> gpurun_out/bench_pdl.err
HMG_PDL=1 timeout 600 python scripts/bench_configs.py --only 0,3 --out gpurun_out/cfg03_pdl.jsonl > gpurun_out/cfg03_pdl.log 2>&1
HMG_PDL=1 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_pdl.log 2>&1; echo exit=$? >> gpurun_out/t_pdl.log
