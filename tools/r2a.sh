set -x
nproc; free -g; lscpu | head -20
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py --config E --steps 3 --warmup 3 > gpurun_out/r2a_benchE.json 2> gpurun_out/r2a_benchE.err
tail -3 gpurun_out/r2a_benchE.err
cat gpurun_out/r2a_benchE.json
