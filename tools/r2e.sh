python -m pytest tests/test_gpu_parity.py -x -q -k "Q_values or end_to_end" 2>&1 | tail -2
python -m pytest tests/test_gpu_fullsize.py -x -q -k "E_sampled" 2>&1 | tail -2
for v in "" "XM_TRSM_SB=256" "XM_GEMM_BK32=1" "XM_TRSM_SB=1024"; do echo "== $v"; env $v XM_VERBOSE=1 python tools/repro_E.py E bb 2>&1 | grep -v "^\s*$" | tail -5; done
