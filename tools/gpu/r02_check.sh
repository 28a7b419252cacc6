mkdir -p gpurun_out
set -x
python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r02_g2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_g2_pytest.log
timeout 900 python bench.py > gpurun_out/r02_g2_bench.json 2> gpurun_out/r02_g2_bench.err; echo "bench rc=$?" >> gpurun_out/r02_g2_bench.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 2 > gpurun_out/r02_g2_ref.json 2> gpurun_out/r02_g2_ref.err; echo "ref rc=$?" >> gpurun_out/r02_g2_ref.err
