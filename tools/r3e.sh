timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 4000 --launch-count 2000 --csv --log-file gpurun_out/r3e_win.csv python tools/imp_solve.py E > gpurun_out/r3e.log 2>&1
python - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/r3e_win.csv')) if len(r)>5 and r[-3]=='gpu__time_duration.sum']
agg=defaultdict(lambda:[0,0.0])
for r in rows:
    n=r[4].split('(')[0]; agg[n][0]+=1; agg[n][1]+=float(r[-1])/1e3
tot=sum(v[1] for v in agg.values())
print(len(rows),'launches', tot/1e3,'ms')
for n,(c,us) in sorted(agg.items(), key=lambda kv:-kv[1][1])[:25]: print(f"{n[:60]:60s} {c:6d} {us/1e3:8.2f} ms {us/c:8.2f} us")
PY
