mkdir -p gpurun_out
for v in ring0 ringy; do
  PNRTE_LIB=variants/$v/libpnrte_b200.so timeout 900 python experiments/ring/ring_probe.py > gpurun_out/r02_ring_$v.jsonl 2> gpurun_out/r02_ring_$v.err
  echo "$v rc=$?"
  cat gpurun_out/r02_ring_$v.jsonl | cut -c1-600
done
timeout 1500 python -m pytest tests/test_gpu_perfcfg.py -m gpu -x -v --timeout 1200 --durations=0 > gpurun_out/r02_perfcfg_pytest.log 2>&1
echo "pytest rc=$?"
tail -n 25 gpurun_out/r02_perfcfg_pytest.log
