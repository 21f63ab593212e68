"""One full, timed oracle solve-to-certificate (build Q → staircase with
Lanczos certificates → round/recover → report) on a BASELINE config, on the
host cores, with the oracle's OWN trajectory counts — the calibration of the
sampled oracle estimate that bench.py's reference arm / cpu_baseline report.

    python tools/oracle_full.py E > profiles/r2_oracle_full_E.json

Counts: every Q·X product (by its column count r) through an ndarray view
that counts __matmul__; Lanczos steps through a wrapper of
lanczos_min_eig.  The oracle's arithmetic is untouched.  Then the same
per-unit samples bench.py takes (oracle HVPs per rank, Lanczos steps) are
timed and the model  T_build + Σ_r n_r·t_hvp(r) + T_lanczos(n_lz) + n_outer·t_outer  is compared with
the measured total."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import xm_oracle as xo  # noqa: E402
from synth.scenes import config_scene  # noqa: E402
import bench  # noqa: E402  (the sampling functions the bench uses)


class CountingQ(np.ndarray):
    counts = {}

    def __matmul__(self, other):
        r = 1 if np.ndim(other) == 1 else int(np.shape(other)[1])
        CountingQ.counts[r] = CountingQ.counts.get(r, 0) + 1
        return np.asarray(self) @ other


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "E"
    sc = config_scene(cfg, seed=0)
    lz = {"steps": 0, "calls": 0}
    orig = xo.lanczos_min_eig

    def counted(*a, **k):
        out = orig(*a, **k)
        lz["steps"] += out[2]
        lz["calls"] += 1
        return out
    xo.lanczos_min_eig = counted
    t0 = time.perf_counter()
    dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
    t_build = time.perf_counter() - t0
    dm.Q = dm.Q.view(CountingQ)
    t1 = time.perf_counter()
    st = xo.staircase(dm, xo.Options())
    t_stair = time.perf_counter() - t1
    t2 = time.perf_counter()
    sol = xo.round_recover(dm, st.Y)
    rep = xo.report(st.cert, sol.rho_hat, dm.normF, 1e-6)
    t_round = time.perf_counter() - t2
    total = time.perf_counter() - t0
    xo.lanczos_min_eig = orig
    dm.Q = np.asarray(dm.Q)
    counts = dict(CountingQ.counts)
    n_lz_products = lz["steps"]
    by_r = {int(r): int(c) for r, c in counts.items()}
    by_r[1] = by_r.get(1, 0) - n_lz_products          # r = 1 products outside Lanczos
    samples = bench.oracle_unit_times(dm, sorted(r for r, c in by_r.items() if c > 0 and r > 1),
                                      lz["steps"])
    model = t_build + sum(by_r[r] * samples["t_hvp"][r] for r in by_r if r > 1 and by_r[r] > 0) \
        + samples["t_lz_total"] + st.outer * samples["t_outer"]
    out = {"config": cfg, "N": sc.N, "M": sc.M, "E": int(sc.E),
           "cores": bench.oracle_threads(), "cpu": bench.cpu_model(),
           "measured_s": {"total": total, "build_Q": t_build, "staircase": t_stair,
                          "round_report": t_round},
           "counts": {"products_by_r": by_r, "lanczos_steps": lz["steps"],
                      "lanczos_calls": lz["calls"], "hvps": st.n_hvp, "spmms": st.n_spmm,
                      "outer": st.outer, "ranks": st.ranks},
           "result": {"f": st.f, "r": st.r, "certified": st.certified,
                      "lambda_min": st.cert.lambda_min, "eta": rep["eta"]},
           "unit_samples": {"t_hvp": {str(k): v for k, v in samples["t_hvp"].items()},
                            "t_lz_total": samples["t_lz_total"], "lz_how": samples["lz_how"],
                            "t_outer": samples["t_outer"]},
           "model_s": model, "model_over_measured": model / total}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
