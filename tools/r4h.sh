OUT=gpurun_out/r4h; mkdir -p $OUT
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_E.csv python tools/imp_solve.py E 1 > $OUT/launch.log 2>&1
python tools/launch_summary.py $OUT/launches_E.csv 0 > $OUT/launches_E_summary.txt 2>&1
rm -f $OUT/launches_E.csv.gz; gzip -k $OUT/launches_E.csv 2>/dev/null; rm -f $OUT/launches_E.csv
tail -3 $OUT/launch.log; head -20 $OUT/launches_E_summary.txt
