mkdir -p gpurun_out
for v in fr2 fr3; do
  PNRTE_LIB=variants/$v/libpnrte_b200.so timeout 900 python experiments/fused_r_pipeline/fuse_probe.py --iters 100 > gpurun_out/r02_fuse3_$v.jsonl 2> gpurun_out/r02_fuse3_$v.err
  echo "$v check rc=$? same=$(grep -c '"same": true' gpurun_out/r02_fuse3_$v.jsonl) diff=$(grep -c '"same": false' gpurun_out/r02_fuse3_$v.jsonl)"
  FUSE_DS=2,3,4,6 PNRTE_LIB=variants/$v/libpnrte_b200.so timeout 900 python experiments/fused_r_pipeline/fuse_probe.py --skip-check --iters 100 >> gpurun_out/r02_fuse3_$v.jsonl 2>> gpurun_out/r02_fuse3_$v.err
  grep '"config"' gpurun_out/r02_fuse3_$v.jsonl | cut -c1-260
  tail -n 2 gpurun_out/r02_fuse3_$v.err
done
