mkdir -p gpurun_out
S=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 --durations=8 > gpurun_out/r02_pytest_gpu_final.log 2>&1
echo "pytest rc=$? $(( $(date +%s) - S )) s"; tail -n 12 gpurun_out/r02_pytest_gpu_final.log
S=$(date +%s)
timeout 1200 python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err
echo "bench rc=$? $(( $(date +%s) - S )) s"; cut -c1-400 gpurun_out/r02_bench_final.json
S=$(date +%s)
timeout 1200 python bench.py --impl reference > gpurun_out/r02_bench_reference_final.json 2> gpurun_out/r02_bench_reference_final.err
echo "ref rc=$? $(( $(date +%s) - S )) s"; cut -c1-400 gpurun_out/r02_bench_reference_final.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 2
