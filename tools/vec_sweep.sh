for v in vec2 scal vec2 scal; do echo "== $v"; PNRTE_LIB=$PWD/variants/$v/libpnrte_b200.so python tools/vec_probe.py --config 4; done
