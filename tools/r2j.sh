python -m pytest tests/test_gpu_parity.py -x -q -k "Q_values or end_to_end_solve_parity" 2>&1 | tail -2
python -m pytest tests/test_gpu_fullsize.py -x -q -k "B_pattern or E_sampled" 2>&1 | tail -2
for c in E B D C; do XM_VERBOSE=1 python tools/repro_E.py $c bb 2>&1 | grep "scatter\|b ok" | tail -2; done
ncu --set full --clock-control none -k regex:clique_scatter_fx --launch-count 1 -o gpurun_out/r2j_scatter_E python tools/repro_E.py E b > /dev/null 2>&1; ls gpurun_out
