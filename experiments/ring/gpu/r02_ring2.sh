mkdir -p gpurun_out
timeout 600 python tools/faithful_probe.py --iters 10 > gpurun_out/r02_faithful_probe.jsonl 2> gpurun_out/r02_faithful_probe.err
echo "faithful rc=$?"; cat gpurun_out/r02_faithful_probe.jsonl
for v in ringwgy ringwg0; do
  PNRTE_LIB=variants/$v/libpnrte_b200.so timeout 600 python experiments/ring/ring_probe.py --rings 1 > gpurun_out/r02_ring_$v.jsonl 2> gpurun_out/r02_ring_$v.err
  echo "$v rc=$?"
  tail -n 1 gpurun_out/r02_ring_$v.jsonl | cut -c1-700
done
export PNRTE_LIB=variants/ringy/libpnrte_b200.so
PNRTE_SEG_RING=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_seg_ring -s 2 -c 2 -o gpurun_out/r02_ring_ncu python tools/profile_apply.py --config 4 --reps 4 > gpurun_out/r02_ring_ncu.log 2>&1
echo "ncu rc=$?"
unset PNRTE_LIB
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 --deselect tests/test_gpu_perfcfg.py::test_fullsize_cfg3_solve_parity > gpurun_out/r02_pytest_gpu_s4.log 2>&1
echo "pytest rc=$?"; tail -n 5 gpurun_out/r02_pytest_gpu_s4.log
