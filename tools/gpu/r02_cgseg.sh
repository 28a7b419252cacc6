mkdir -p gpurun_out
rm -f gpurun_out/r02_cgseg_*.log
python -m pytest tests/test_gpu_cgseg.py -q > gpurun_out/r02_cgseg_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_cgseg_pytest.log
python tools/iter_probe.py --config 2 --iters 200 >> gpurun_out/r02_cgseg_iter.log 2>&1
PNRTE_CGSEG_MAX=0 python tools/iter_probe.py --config 2 --iters 200 >> gpurun_out/r02_cgseg_iter.log 2>&1
python tools/ttr.py --configs 1,2 > gpurun_out/r02_cgseg_ttr.log 2>&1
