# rebuild with each build-environment variant (";"-separated in $VARIANTS, e.g.
# "PNRTE_NVCC_FLAGS=-DPN_SEG_PF=222;PNRTE_RED_SEQ=1"; an empty entry is the
# default build) and time the config-4 / config-3 applies, plain and with
# fused reductions, plus the config-3 / config-4 CG iteration
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for V in "${VS[@]}"; do
  env $V python -c "from paper_1807_00410_b200 import build; build.build(force=True)" > /dev/null 2>&1 || echo "build fail [$V]"
  echo "VARIANT=[$V]"
  for w in 0 2 1; do python tools/profile_apply.py --config 4 --what $w --reps 10; python tools/profile_apply.py --config 3 --what $w --reps 50; done
done
