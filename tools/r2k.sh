python -m pytest tests/test_gpu_parity.py -x -q -k "Q_values" 2>&1 | tail -1
for v in "" "XM_SCATTER_CFG=768" "XM_SCATTER_CFG=256"; do echo "== $v"; for c in E D; do env $v XM_VERBOSE=1 python tools/repro_E.py $c bb 2>&1 | grep "scatter" | tail -1; done; done
