python -m pytest tests/test_gpu_parity.py -x -q -k "Q_values or end_to_end" 2>&1 | tail -2
python -m pytest tests/test_gpu_fullsize.py -x -q -k "B_pattern or E_sampled" 2>&1 | tail -2
XM_VERBOSE=1 python tools/repro_E.py E bb 2>&1 | grep -v "^\s*$" | tail -7
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches_buildE.csv python tools/repro_E.py E b > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2d_launches_buildE.csv 2>&1 | head -30
