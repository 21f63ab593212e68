python -m pytest tests/test_gpu_tcg.py tests/test_gpu_parity.py tests/test_gpu_xm2.py -q -x 2>&1 | tail -3
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_run.py > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|SANITIZE_RUN_OK|RACECHECK SUMMARY" gpurun_out/r2_sanitize_$tool.log | tail -3
done
timeout 900 python bench.py --config B --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2r_benchB.json 2>gpurun_out/r2r_benchB.err; tail -2 gpurun_out/r2r_benchB.err; cat gpurun_out/r2r_benchB.json
