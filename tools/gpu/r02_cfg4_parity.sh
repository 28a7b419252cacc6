mkdir -p gpurun_out
timeout 200 python tools/cfg4_solve_parity.py --config 4 --n 32 --out gpurun_out/r02_cfg4_solve_parity_n32.json 2>&1 | tail -n 3 | cut -c1-600
timeout 7000 python tools/cfg4_solve_parity.py > gpurun_out/r02_cfg4_solve_parity.log 2>&1
echo "rc=$?"; tail -n 3 gpurun_out/r02_cfg4_solve_parity.log | cut -c1-900
