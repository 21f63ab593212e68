# A/B of the Q·V kernels on B200: lower-triangle vs full-row at
# configs B and E, and the lower-triangle kernel with its compute / finish
# switched off (stream-only bound).  Usage: bash tools/exp_sym.sh [cfgs]
set -e
CFGS=${CFGS:-"B E"}
python -m paper_2502_04640_b200.build --force > /dev/null
for C in $CFGS; do
  XM_FORCE_SYM=1 python tools/spmm_bench.py $C 1 3 4 5
  XM_NO_SYM=1 python tools/spmm_bench.py $C 1 3 4
done
for F in "-DXM_EXP_NOFINISH" "-DXM_EXP_NOCOMPUTE -DXM_EXP_NOFINISH"; do
  XM_NVCC_EXTRA="$F" python -m paper_2502_04640_b200.build --force > /dev/null
  for C in $CFGS; do XM_FORCE_SYM=1 XM_NVCC_EXTRA="$F" python tools/spmm_bench.py $C 1 3; done
done
python -m paper_2502_04640_b200.build --force > /dev/null
