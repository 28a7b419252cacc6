for S in ${SUBS:-1 2 4 8}; do
  PNRTE_NVCC_FLAGS="-DPN_CSR_SUB=$S" python -c "from paper_1807_00410_b200 import build; build.build(force=True)" > /dev/null 2>&1 || echo "build fail $S"
  echo "SUB=$S"; timeout 200 python tools/widened_probe.py 2>&1 | grep "device CSR\|CDA" | cut -c1-200
done
