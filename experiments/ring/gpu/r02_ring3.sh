mkdir -p gpurun_out
for v in ringy ring0; do
  PNRTE_LIB=variants/$v/libpnrte_b200.so timeout 600 python experiments/ring/ring_probe.py --rings 1 > gpurun_out/r02_ring3_$v.jsonl 2> gpurun_out/r02_ring3_$v.err
  echo "$v rc=$?"
  grep -c '"same": true' gpurun_out/r02_ring3_$v.jsonl; grep '"same": false' gpurun_out/r02_ring3_$v.jsonl
  tail -n 1 gpurun_out/r02_ring3_$v.jsonl | cut -c1-700
  tail -n 3 gpurun_out/r02_ring3_$v.err
done
export PNRTE_LIB=variants/ringy/libpnrte_b200.so
PNRTE_SEG_RING=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_seg_ring -s 2 -c 2 -o gpurun_out/r02_ring3_ncu python tools/profile_apply.py --config 4 --reps 4 > gpurun_out/r02_ring3_ncu.log 2>&1
echo "ncu rc=$?"
unset PNRTE_LIB
timeout 900 python -m pytest tests/test_gpu_perfcfg.py -m gpu -x -v -s --timeout 800 -k fullsize_cfg3 > gpurun_out/r02_cfg3_full_pytest.log 2>&1
echo "pytest rc=$?"; tail -n 8 gpurun_out/r02_cfg3_full_pytest.log
