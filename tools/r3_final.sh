set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2000 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 1200 python bench.py > gpurun_out/r3f_bench_E.json 2> gpurun_out/r3f_bench_E.err; tail -2 gpurun_out/r3f_bench_E.err
timeout 600 python bench.py --config B --no-cpu-baseline > gpurun_out/r3f_bench_B.json 2> gpurun_out/r3f_bench_B.err
