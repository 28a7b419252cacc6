mkdir -p gpurun_out
timeout 600 python experiments/ring/ring_probe.py --rings 1 > gpurun_out/r02_ring6.jsonl 2> gpurun_out/r02_ring6.err
echo "ring rc=$?"
grep -c '"same": true' gpurun_out/r02_ring6.jsonl; grep '"same": false' gpurun_out/r02_ring6.jsonl
tail -n 1 gpurun_out/r02_ring6.jsonl | cut -c1-700
tail -n 3 gpurun_out/r02_ring6.err
timeout 300 python experiments/ring/ring_probe.py --config 3 --skip-check --rings 1 2>&1 | cut -c1-400
PNRTE_SEG_RING=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_seg_ring -s 2 -c 1 -o gpurun_out/r02_ring6_ncu python tools/profile_apply.py --config 4 --reps 4 > gpurun_out/r02_ring6_ncu.log 2>&1
echo "ncu ring rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_seg -s 2 -c 1 -o gpurun_out/r02_grid_ncu python tools/profile_apply.py --config 4 --reps 4 > gpurun_out/r02_grid_ncu.log 2>&1
echo "ncu grid rc=$?"
