set -x
OUT=gpurun_out/r4e; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 2000 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $OUT/gpu_tests.txt; cat $OUT/gpu_tests.txt
timeout 1200 python bench.py > $OUT/bench_E.json 2> $OUT/bench_E.err; tail -2 $OUT/bench_E.err; cat $OUT/bench_E.json
timeout 600 python bench.py --config B --no-cpu-baseline > $OUT/bench_B.json 2> $OUT/bench_B.err; cat $OUT/bench_B.json
