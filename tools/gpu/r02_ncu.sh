mkdir -p gpurun_out
CMD="python bench.py --steps 4 --warmup 3 --sustain-s 0.05 --skip-ttr --skip-ttr4 --skip-e2e --skip-cpu --skip-others --skip-paper"
$CMD > gpurun_out/r02_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_bench.csv $CMD > gpurun_out/r02_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_seg -s 3 -c 2 -o gpurun_out/r02_apply $CMD > gpurun_out/r02_ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/r02_ncu_full.log
