mkdir -p gpurun_out
python -c "import pynvml" 2>/dev/null || echo "no pynvml"
python tools/power_probe.py --config 4 > gpurun_out/r02_power_cfg4.jsonl 2> gpurun_out/r02_power_cfg4.err
python tools/power_probe.py --config 2 > gpurun_out/r02_power_cfg2.jsonl 2> gpurun_out/r02_power_cfg2.err
python tools/iter_probe.py --config 2 --iters 200 > gpurun_out/r02_iter_cfg2.log 2>&1
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python tools/sanitize_probe.py > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r02_sanitize_$tool.log
done
