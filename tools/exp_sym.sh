set -e
python -m paper_2502_04640_b200.build --force > /dev/null
XM_FORCE_SYM=1 python tools/spmm_bench.py B 1 3
XM_NO_SYM=1 python tools/spmm_bench.py B 1 3
for F in "-DXM_EXP_NOFINISH" "-DXM_EXP_NOCOMPUTE -DXM_EXP_NOFINISH" "-DXM_EXP_NOCOMPUTE"; do
  XM_NVCC_EXTRA="$F" python -m paper_2502_04640_b200.build --force > /dev/null
  XM_FORCE_SYM=1 XM_NVCC_EXTRA="$F" python tools/spmm_bench.py B 1 3
done
python -m paper_2502_04640_b200.build --force > /dev/null
XM_FORCE_SYM=1 python tools/spmm_bench.py E 3
XM_NO_SYM=1 python tools/spmm_bench.py E 3
