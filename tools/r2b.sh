# H5 on the DMMA kernel: Q parity (small scenes, B, sampled E) + build phases at B, E
python -m pytest tests/test_gpu_parity.py -x -q -k "Q_values or end_to_end" 2>&1 | tail -3
python -m pytest tests/test_gpu_fullsize.py -x -q -k "B_pattern or E_sampled" 2>&1 | tail -3
for cfg in B E; do XM_VERBOSE=1 python tools/repro_E.py $cfg bb 2>&1 | grep -v "^\s*$" | tail -14; done
