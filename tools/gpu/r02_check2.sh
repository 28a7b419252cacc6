mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=12 > gpurun_out/r02_c2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_c2_pytest.log
python bench.py --weak --steps 10 --warmup 3 > gpurun_out/r02_c2_weak.json 2> gpurun_out/r02_c2_weak.err; echo "rc=$?" >> gpurun_out/r02_c2_weak.err
python bench.py --cfg5 --cfg5-n 256 --steps 10 --warmup 3 --skip-ttr4 --skip-e2e --skip-cpu --skip-others --skip-paper --skip-ttr > gpurun_out/r02_c2_cfg5val.json 2> gpurun_out/r02_c2_cfg5val.err; echo "rc=$?" >> gpurun_out/r02_c2_cfg5val.err
