mkdir -p gpurun_out
for v in r5y0 r6y0 r6y1 r5y1; do
  PNRTE_LIB=variants/$v/libpnrte_b200.so timeout 400 python experiments/ring/ring_probe.py --rings 1 --skip-check > gpurun_out/r02_ring5_$v.jsonl 2> gpurun_out/r02_ring5_$v.err
  echo "$v rc=$?"
  tail -n 1 gpurun_out/r02_ring5_$v.jsonl | cut -c1-330
done
for v in ringy r6y1; do
  PNRTE_LIB=variants/$v/libpnrte_b200.so timeout 400 python experiments/ring/ring_probe.py --config 3 --skip-check > gpurun_out/r02_ring5_cfg3_$v.jsonl 2> gpurun_out/r02_ring5_cfg3_$v.err
  echo "cfg3 $v rc=$?"
  cut -c1-330 gpurun_out/r02_ring5_cfg3_$v.jsonl
done
timeout 900 python -m pytest tests/test_gpu_perfcfg.py -m gpu -x -v -s --timeout 800 -k fullsize_cfg3 > gpurun_out/r02_cfg3_full_pytest.log 2>&1
echo "pytest rc=$?"; tail -n 4 gpurun_out/r02_cfg3_full_pytest.log
