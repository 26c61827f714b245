mkdir -p gpurun_out
python scripts/probe.py --config 1 --iters 2 > gpurun_out/probe1.log 2>&1 || exit 1
python scripts/probe.py --config 3 --iters 2 > gpurun_out/probe3.log 2>&1 || exit 1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_stored_op2d_pair|k_rb2d_march2|k_fine_op2d_pair|k_fine_op|k_restrict_pair|k_prolong_block" -c 12 -o /tmp/n1 python scripts/probe.py --config 1 --iters 2 > gpurun_out/ncu1.log 2>&1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_fine_op3d_z|k_stored_op|k_vanka_stencil|k_fine_op" -c 10 -o /tmp/n3 python scripts/probe.py --config 3 --iters 2 > gpurun_out/ncu3.log 2>&1
for f in n1 n3; do
  ncu -i /tmp/$f.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/${f}_raw.csv.gz
  ncu -i /tmp/$f.ncu-rep --page details --csv 2>/dev/null | gzip > gpurun_out/${f}_details.csv.gz

done
ls -la gpurun_out
