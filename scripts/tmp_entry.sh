( time timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" ) > gpurun_out/smoke.log 2>&1
( time timeout 900 python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/ref_default.json 2> gpurun_out/ref_default.err
