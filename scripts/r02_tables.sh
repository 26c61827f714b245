mkdir -p gpurun_out
timeout 1500 python scripts/paper_tables.py --out gpurun_out/r02_paper_tables.json > gpurun_out/tables.log 2>&1
timeout 1200 python scripts/damping_search.py --out gpurun_out/r02_damping_search.json > gpurun_out/damping.log 2>&1
