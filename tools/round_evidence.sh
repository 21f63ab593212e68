#!/bin/bash
# One GPU call that produces a round's measurement evidence under gpurun_out/:
# bench lines (xm arm B with cpu_baseline + e2e, reference arm B, xm arm E),
# the ncu launch list of the bench command, `ncu --set full` captures of the
# dominant kernels (k_tcg_persist_sym at B; k_spmm_sym at E, r = 3 and 4).
set -x
OUT=gpurun_out/${TAG:-r1}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/gpu.txt
timeout 900 python bench.py > $OUT/bench_B.json 2> $OUT/bench_B.err
timeout 900 python bench.py --impl reference > $OUT/bench_ref_B.json 2> $OUT/bench_ref_B.err
timeout 900 python bench.py --config E --no-cpu-baseline > $OUT/bench_E.json 2> $OUT/bench_E.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_B.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > $OUT/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tcg_persist \
  --launch-skip ${SKIP:-30} --launch-count ${COUNT:-2} -o $OUT/ncu_full_B -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
TAG=${TAG:-r1} timeout 1200 bash tools/exp_sym_ncu.sh
ls -la $OUT
XM_PHASES=1 timeout 120 python tools/repro_E.py B bs 2>&1 | grep -v "^\s*$"
