# rebuild with each build variant and time the config-4 / config-3 applies
# (plain and with fused reductions) and CG iterations.  $VARIANTS: ";"-separated
# entries, each "ENV=VALUE" assignments separated by spaces, where commas inside a
# value stand for spaces (e.g. "PNRTE_NVCC_FLAGS=-DPN_SEG_QUAD=2,-DPN_SEG_QUAD_MINB=3");
# an empty entry is the default build.  $CONFIGS: configs to time (default "4 3").
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for V in "${VS[@]}"; do
  ARGS=()
  for a in $V; do ARGS+=("${a//,/ }"); done
  env "${ARGS[@]}" python -c "from paper_1807_00410_b200 import build; build.build(force=True)" > /dev/null 2>&1 || echo "build fail [$V]"
  echo "VARIANT=[$V]"
  for w in 0 2 1; do
    for c in ${CONFIGS:-4 3}; do
      python tools/profile_apply.py --config $c --what $w --reps $([ "$c" = 4 ] && echo 10 || echo 50)
    done
  done
done
