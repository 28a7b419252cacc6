mkdir -p gpurun_out
for v in base priv base priv; do PNRTE_LIB=variants/$v/libpnrte_b200.so python tools/variant_probe.py $v >> gpurun_out/r02_ab1.jsonl 2>> gpurun_out/r02_ab1.err; done
python tools/e2e_probe.py > gpurun_out/r02_e2e_probe.jsonl 2> gpurun_out/r02_e2e_probe.err
