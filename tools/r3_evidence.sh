#!/bin/bash
# Round-3 (this round's second half) evidence for the matrix-free headline at E:
# bench line (cpu_baseline + e2e + other_mode), reference arm, the ncu launch list of
# one bench step, and an `ncu --set full` capture of one matrix-free product's kernels.
set -x
OUT=gpurun_out/${TAG:-r3}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.limit --format=csv > $OUT/gpu.txt
timeout 1200 python bench.py > $OUT/bench_E.json 2> $OUT/bench_E.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref_E.json 2> $OUT/bench_ref_E.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_E.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-other-mode --mode implicit \
  > $OUT/ncu_launch.log 2>&1
python tools/launch_summary.py $OUT/launches_E.csv 3 > $OUT/launches_E_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'k_imp_lm_mean|k_imp_fr_b|k_spmm_sym|k_imp_lm_p|k_imp_fr_out' \
  --launch-skip 25 --launch-count 10 -o $OUT/ncu_full_imp_E -f python tools/imp_prof.py E > $OUT/ncu_full.log 2>&1
ls -la $OUT
