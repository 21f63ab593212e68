set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 600 python bench.py > gpurun_out/r3a_bench_E.json 2> gpurun_out/r3a_bench_E.err; tail -3 gpurun_out/r3a_bench_E.err
cat gpurun_out/r3a_bench_E.json
