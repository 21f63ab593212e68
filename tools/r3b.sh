timeout 900 python -m pytest tests/test_gpu_implicit.py -q -x 2>&1 | tail -15
timeout 600 python - <<'PY' 2>&1 | tail -8
import sys, time
sys.path.insert(0, '.')
from paper_2502_04640_b200 import xm
from synth.scenes import config_scene
sc = config_scene("E")
for imp in (1, 1):
    with xm.Context(implicit_q=imp) as ctx:
        t = time.time(); ctx.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w); tb = time.time() - t
        t = time.time(); s, info = ctx.solve(); ts = time.time() - t
        t = time.time(); cert = ctx.certify(); tc = time.time() - t
        print("implicit", imp, "build %.3f solve %.3f cert %.3f" % (tb, ts, tc), "hvps", info["hvps"], "spmms", info["spmms"], "r", info["r"], "eta", cert["eta"], flush=True)
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:'k_imp_|k_spmm_sym' --launch-skip 20 --launch-count 10 python tools/imp_prof.py E 2>&1 | grep -E "k_imp|k_spmm|duration|dram__bytes" | head -40
