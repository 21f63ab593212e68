timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_E2.csv python tools/imp_solve.py E 1 > gpurun_out/r2b_launch.log 2>&1
python tools/launch_summary.py gpurun_out/r2b_launches_E2.csv 0 > gpurun_out/r2b_launches_E2_summary.txt 2>&1
tail -3 gpurun_out/r2b_launch.log
