XM_IMP_U="8,16,16,8" timeout 600 python -m pytest tests/test_gpu_implicit.py -q -x 2>&1 | tail -1
for v in "0,0,0,0" "8,8,8,4" "8,16,16,8" "16,16,16,8" "16,16,16,4" "2,2,2,2"; do
  echo "=== U [$v]"
  XM_IMP_U=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_imp_' --launch-skip 16 --launch-count 4 python tools/imp_prof.py E 2>&1 | grep -E "^\s+void|duration" | sed -E 's/\(int.*//; s/.*unnamed>:://' | paste - - | awk '{printf "%s %s  ", $1, $NF} END {print ""}'
done
