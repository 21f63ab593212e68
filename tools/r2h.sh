python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; tail -3 gpurun_out/r2h_bench.err; cat gpurun_out/r2h_bench.json
