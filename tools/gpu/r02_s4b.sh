mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_solver.py -m gpu -x -q --timeout 300 -k "nccl or solve_host or end_to_end" > gpurun_out/r02_pytest_new.log 2>&1
echo "pytest rc=$?"; tail -n 15 gpurun_out/r02_pytest_new.log
timeout 900 python tools/ttr.py --configs 1,2,3,4 --jacobi > gpurun_out/r02_ttr_jacobi.jsonl 2> gpurun_out/r02_ttr_jacobi.err
echo "ttr rc=$?"; cat gpurun_out/r02_ttr_jacobi.jsonl; tail -n 3 gpurun_out/r02_ttr_jacobi.err
