timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2bb_benchE.json 2> gpurun_out/r2bb_benchE.err; tail -3 gpurun_out/r2bb_benchE.err; cat gpurun_out/r2bb_benchE.json
