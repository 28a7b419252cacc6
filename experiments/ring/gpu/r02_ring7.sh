mkdir -p gpurun_out
for v in c6e3 c4e4 c4e3; do
  PNRTE_LIB=variants/$v/libpnrte_b200.so timeout 400 python experiments/ring/ring_probe.py --rings 1 --skip-check > gpurun_out/r02_ring7_$v.jsonl 2> gpurun_out/r02_ring7_$v.err
  echo "$v rc=$?"
  tail -n 1 gpurun_out/r02_ring7_$v.jsonl | cut -c1-330
  PNRTE_LIB=variants/$v/libpnrte_b200.so timeout 300 python experiments/ring/ring_probe.py --config 3 --skip-check --rings 1 2>&1 | cut -c1-330
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_seg -s 2 -c 1 -o gpurun_out/r02_grid_ncu python tools/profile_apply.py --config 4 --reps 4 > gpurun_out/r02_grid_ncu.log 2>&1
echo "ncu grid rc=$?"
