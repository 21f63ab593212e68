timeout 600 python -m pytest tests/test_gpu_edge_cases.py -q -x -k implicit 2>&1 | grep -E 'assert|Error|passed|failed' | head -20
for v in "XM_IMP_NONE=1" "XM_IMP_LMRO=1 XM_IMP_FRCO=1"; do
  echo "=== variant [$v]"
  env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_imp_' --launch-skip 16 --launch-count 8 python tools/imp_prof.py E 2>&1 | grep -E "^\s+void|duration" | sed -E 's/\(int.*//; s/.*unnamed>:://' | paste - - | awk '{print $1, $NF}'
done
