timeout 600 python -m pytest tests/test_gpu_edge_cases.py -q -x 2>&1 | tail -3
# A/B: record-based pass variants; conditional-graph tCG loop
for v in "" "XM_IMP_LMRO=1 XM_IMP_FRCO=1"; do
  echo "=== variant [$v]"
  env $v timeout 600 python -m pytest tests/test_gpu_implicit.py -q -x 2>&1 | tail -2
  env $v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:'k_imp_' --launch-skip 16 --launch-count 8 python tools/imp_prof.py E 2>&1 | grep -E "k_imp|duration" | paste - - | awk '{print $2, $NF}' | sed -E 's/\(int.*//' 
done
for v in "XM_NO_COND_GRAPH=1" "" "XM_IMP_LMRO=1 XM_IMP_FRCO=1"; do
  echo "=== solve [$v]"
  env $v timeout 300 python tools/imp_solve.py E 3 2>&1 | grep -E '^build|rror' 
done
