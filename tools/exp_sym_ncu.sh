# ncu --set full of one k_spmm_sym launch on config E at r=3 and r=4
# (tools/spmm_bench.py: 5 warm-up products, then 50 timed).
OUT=gpurun_out/${TAG:-sym}
mkdir -p $OUT
for r in ${RS:-3 4}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_sym \
    --launch-skip 5 --launch-count 1 -o $OUT/ncu_sym_E_r$r -f \
    env XM_FORCE_SYM=1 python tools/spmm_bench.py ${CFG:-E} $r > $OUT/ncu_sym_r$r.log 2>&1
done
