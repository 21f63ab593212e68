python -m pytest tests/test_gpu_xm2.py -q -x -k restoration 2>&1 | grep -E "^E |assert|Error" | head -30
python -m pytest tests/test_gpu_scale_reg.py tests/test_gpu_edge_cases.py -q 2>&1 | tail -3
for v in "" "XM_GEMM_TILE=w16"; do echo "== $v"; env $v XM_VERBOSE=1 python tools/repro_E.py E bb 2>&1 | grep -v "^\s*$" | grep "cholesky\|trsm\|syrk\|scatter" | tail -4; done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2_sanitize_memcheck.log 2>&1; tail -5 gpurun_out/r2_sanitize_memcheck.log
