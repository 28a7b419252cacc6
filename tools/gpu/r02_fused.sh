mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r02_fused_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_fused_pytest.log
for c in 2 3 4; do python tools/iter_probe.py --config $c --iters 100 >> gpurun_out/r02_fused_iter.log 2>&1; done
