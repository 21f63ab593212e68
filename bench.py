#!/usr/bin/env python
"""Benchmark of the XM hot path on B200 (BASELINE.json metric:
"solve-to-certificate seconds & HVP/s; SpMM HBM GB/s vs peak").

One STEP = one pass of the whole hot path (SURVEY §8(a) H1–H13) over one
synthetic view graph: xm_build_Q → xm_solve (staircase, every rank certified
with Lanczos) → xm_certify → xm_round_recover.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config B] [--impl xm|reference]

Multi-GPU (N > 1) is launched by torchrun; Q rows are sharded across ranks
and the library all-gathers Q·V shards with NCCL (strong scaling: the total
work is fixed).  Timing: CUDA events on the library's stream (torch's current
stream is passed to xm_create), barrier + synchronize around the K timed steps,
max over ranks.  Inputs (Q is 288 MB at config B, 7.4 GB at E) are larger than
the 126 MB L2, so no explicit flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback ("of fallback")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "spmm_traffic.json")
METRIC = "solve_to_certificate_s"


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.gpu_idle,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        try:
            rows = [l.strip().split(", ") for l in open(self.path) if l.strip()]
        except Exception:
            rows = []
        names = ["gpu_idle", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        sm, mx, reasons = [], 0.0, set()
        for r in rows:
            if len(r) < 7:
                continue
            try:
                cur, m = float(r[0]), float(r[1])
            except ValueError:
                continue
            mx = max(mx, m)
            act = {nm for nm, v in zip(names, r[2:7]) if v.strip().lower() == "active"}
            if "gpu_idle" not in act:
                sm.append(cur)
            reasons |= act - {"gpu_idle"}
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ----------------------------------------------------------------------------- oracle timing
# The oracle (reference arm, cpu_baseline) is timed as it stands on this
# host's cores.  Its full solve at config E takes ~10 min, so a bench run
# times: the oracle's FULL Q build (once), plus bounded samples of its unit
# operations (oracle HVPs at each rank the oracle's own trajectory visits,
# oracle Lanczos steps), scaled by the counts of the oracle's OWN full
# trajectory (profiles/r2_oracle_full_<cfg>.json, written by
# tools/oracle_full.py, which also times the full solve and records how close
# this model comes to it).  The value is labelled an estimate.  bench.py never
# writes tracked files.

def oracle_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_counts(cfg):
    path = os.path.join(ROOT, "profiles", f"r2_oracle_full_{cfg}.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, os.path.relpath(path, ROOT)
    except Exception:
        return None, None


def oracle_unit_times(dm, ranks, n_lanczos, n_hvp=4):
    """Per-unit oracle times on the full-size Q: one oracle Riemannian HVP
    (xo.hess: Q·V + projection) at a random feasible Y of rank r, for each r;
    the O(n·r) work of one outer TR iteration (retraction + gradient); and the
    oracle's Lanczos run of n_lanczos steps (its full re-orthogonalisation
    makes step k cost a + b·k): timed in full when n_lanczos ≤ 256, else from
    two timed runs of 64 and 256 steps, T(k) = a·k + b·k²/2 fitted and
    evaluated at n_lanczos."""
    import numpy as np
    from oracle import xm_oracle as xo
    from synth.scenes import random_factor, random_tangent_ambient
    Q = np.asarray(dm.Q)
    N = dm.N
    t_hvp = {}
    for r in ranks:
        Y = random_factor(N, r, 1)
        g, Lam = xo.rgrad(Y, Q @ Y)
        V = xo.project(Y, random_tangent_ambient(N, r, 2))
        t0 = time.perf_counter()
        for _ in range(n_hvp):
            xo.hess(Q, Y, Lam, V)
        t_hvp[r] = (time.perf_counter() - t0) / n_hvp
    Y = random_factor(N, 3, 1)
    QY = Q @ Y
    _, Lam = xo.rgrad(Y, QY)
    V = 1e-3 * xo.project(Y, random_tangent_ambient(N, 3, 3))
    t0 = time.perf_counter()
    for _ in range(n_hvp):                   # the O(n·r) work of one outer TR iteration
        xo.retract(Y, V)
        xo.rgrad(Y, QY)
    t_outer = (time.perf_counter() - t0) / n_hvp

    def apply_Z(x):
        X = x.reshape(-1, 1)
        return (Q @ X - xo.block_apply(Lam, X)).ravel()

    def lz_time(k):
        t0 = time.perf_counter()
        xo.lanczos_min_eig(apply_Z, dm.n, 0.0, max_steps=k)
        return time.perf_counter() - t0
    if n_lanczos <= 256:
        t_lz_total, how = (lz_time(n_lanczos) if n_lanczos > 0 else 0.0), f"{n_lanczos} steps timed"
    else:
        k1, k2 = 64, 256
        T1, T2 = lz_time(k1), lz_time(k2)
        b = max(0.0, 2.0 * (T2 / k2 - T1 / k1) / (k2 - k1))
        a = T1 / k1 - b * k1 / 2
        t_lz_total = a * n_lanczos + b * n_lanczos * n_lanczos / 2
        how = (f"{k1} and {k2} steps timed ({T1:.2f} s, {T2:.2f} s), a·k + b·k²/2 at "
               f"k = {n_lanczos}")
    return {"t_hvp": t_hvp, "t_outer": t_outer, "t_lz_total": t_lz_total, "lz_how": how}


class OracleEstimate:
    """Oracle solve-to-certificate time on this host: the measured full Q
    build + sampled unit times × the oracle trajectory's own counts."""

    def __init__(self, scene, cfg):
        self.sc, self.cfg = scene, cfg
        self.full, self.src = oracle_counts(cfg)
        self.dm = None
        self.t_build = None

    def available(self):
        return self.full is not None

    def step(self, n_hvp=4):
        from oracle import xm_oracle as xo
        sc = self.sc
        if self.dm is None:
            t0 = time.perf_counter()
            self.dm = xo.build_Q(sc.N, sc.M, sc.frame, sc.landmark, sc.pts, sc.w)
            self.t_build = time.perf_counter() - t0
        c = self.full["counts"]
        by_r = {int(r): int(v) for r, v in c["products_by_r"].items() if int(r) > 1 and int(v) > 0}
        u = oracle_unit_times(self.dm, sorted(by_r), c["lanczos_steps"], n_hvp)
        est = (self.t_build + sum(by_r[r] * u["t_hvp"][r] for r in by_r)
               + u["t_lz_total"] + c["outer"] * u["t_outer"])
        sample = (f"oracle build_Q timed in full on this workload ({self.t_build:.1f} s, once) + "
                  f"{n_hvp} oracle HVPs per rank {sorted(by_r)} ("
                  + ", ".join(f"r={r}: {u['t_hvp'][r] * 1e3:.0f} ms" for r in sorted(by_r))
                  + f") + the oracle's Lanczos ({u['lz_how']}; {u['t_lz_total']:.1f} s) + {n_hvp} "
                  f"retraction+gradient passes ({u['t_outer'] * 1e3:.0f} ms each), scaled by the "
                  f"oracle's own trajectory counts ({sum(by_r.values())} products, "
                  f"{c['lanczos_steps']} Lanczos steps, {c['outer']} outer iterations; {self.src}, "
                  f"whose full timed oracle run took "
                  f"{self.full['measured_s']['total']:.0f} s with this model at "
                  f"{self.full['model_over_measured']:.3f}x)")
        return est, sample


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    _, rank, _ = dist_env()
    if rank != 0:
        return 0
    from synth.scenes import CONFIG_DESCRIPTIONS, config_scene
    sc = config_scene(args.config, seed=args.seed)
    est = OracleEstimate(sc, args.config)
    if not est.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          f"no oracle trajectory counts for config {args.config} "
                          f"(run tools/oracle_full.py {args.config})"}), flush=True)
        return 0
    times = []
    sample = ""
    for i in range(args.warmup + args.steps):
        v, sample = est.step(n_hvp=2 if i < args.warmup else 4)
        if i >= args.warmup:
            times.append(v)
    v = sum(times) / len(times)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config {args.config}: {CONFIG_DESCRIPTIONS[args.config]}",
                       "N": sc.N, "M": sc.M, "E": sc.E, "seed": args.seed,
                       "counts_source": est.src + " (the oracle's own full trajectory)"},
            "cpu_baseline": {"value": v, "unit": "s", "cores": oracle_threads(), "kind": "oracle",
                             "estimate": True, "cpu": cpu_model(), "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- multi-rank plumbing
def dist_env():
    """(world, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def share_id(dist, rank: int, make):
    """Rank 0 calls make() (the 128-byte ncclUniqueId); every rank returns it."""
    obj = [make() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(dist, x: float, device) -> float:
    """Device-timed numbers are reported as the max over ranks."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- xm arm
def dense_bytes(N: int, r: int) -> float:
    """Algorithmic bytes of one lower-triangle Q·V product."""
    n = 3 * N
    return 8.0 * n * (n + 1) / 2 + 16.0 * n * r


def implicit_bytes(N: int, E: int, r: int) -> float:
    """Algorithmic bytes of one matrix-free Q·V product (implicit_alg_bytes)."""
    m = N - 1
    return 80.0 * E + 8.0 * m * (m + 1) / 2 + 16.0 * 3 * N * r


def pick_implicit(N: int, E: int, world: int) -> bool:
    """--mode auto: the mode with the smaller modelled time per product — the
    dense band streams 1/world of the lower triangle at ≈ 6.1 TB/s plus ONE
    all-reduce; the matrix-free product moves 1/world of its bytes at the
    measured ≈ 2.85 TB/s plus FIVE all-reduces (≈ 20 µs each assumed, 1 MB over
    NVLink).  E: matrix-free on 1 and 2 GPUs, dense band at 4 and 8; B, C, D: dense."""
    ar = 20e-6
    t_dense = dense_bytes(N, 3) / world / 6.1e12 + (ar if world > 1 else 0.0)
    t_imp = implicit_bytes(N, E, 3) / world / 2.85e12 + 15e-6 + (5 * ar if world > 1 else 0.0)
    return t_imp < t_dense  # + 15 µs: five dependent launches per matrix-free product


def roofline_pass(ctx, step, dev_in, out_dev, steps, barrier):
    """K steps with CUDA events around every Q·V product (event records inside
    the graphs add a few µs per launch, so timed regions run without them)."""
    import torch
    ctx.set_profile(True)
    step(dev_in, out_dev)                    # recapture the graphs with event nodes
    torch.cuda.synchronize()
    ctx.reset_stats()
    barrier()
    for _ in range(steps):
        step(dev_in, out_dev)
    torch.cuda.synchronize()
    barrier()
    pstats = ctx.stats()
    ctx.set_profile(False)
    return pstats


def roofline_obj(pstats, kernel, traffic, step_ms, steps):
    ms_per = pstats["spmm_ms"] / max(pstats["spmm_timed"], 1)
    bytes_per = pstats["spmm_alg_bytes"] / max(pstats["spmm_timed"], 1)
    achieved = bytes_per / (ms_per / 1e3) / 1e9 if pstats["spmm_timed"] else None
    peak, peak_kind = hbm_peak()
    return {"kernel": kernel, "bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "alg_bytes_per_launch": bytes_per, "launch_ms": ms_per, "launches": pstats["spmm_timed"],
            "share_of_step": pstats["spmm_ms"] / (step_ms * steps) if step_ms > 0 else None,
            "timing": "CUDA events around every Q·V product (persistent tCG: per launch ÷ its "
                      "iterations; graph replays past a tCG stop excluded), on the library's stream, "
                      "over a second run of min(K, 5) steps"}


def traffic_of(key):
    try:
        with open(TRAFFIC_FILE) as f:
            return json.load(f).get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


KERNEL_DENSE_B = ("k_tcg_persist_sym (lower-triangle Q stream, timed per tCG iteration incl. its "
                  "barriers and camera update) + k_spmm_sym (other products)")
KERNEL_DENSE = "k_spmm_sym (lower-triangle Q stream, every product incl. the tCG HVP)"
KERNEL_IMPLICIT = ("matrix-free Q·V product, timed as one unit: k_imp_vt, k_imp_lm_mean, k_imp_fr_b, "
                   "k_spmm_sym on the lower triangle of K̄⁻¹, k_imp_lm_p, k_imp_fr_out")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="E", choices=list("ABCDE"))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="xm", choices=["xm", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other-mode", action="store_true",
                    help="skip the measurement of the other product mode (profiling runs)")
    ap.add_argument("--mode", default="auto", choices=["auto", "dense", "implicit"],
                    help="headline product mode: dense Q, the matrix-free NEXT-1 products, or auto "
                         "(default: matrix-free on one GPU when its bytes per product are under half "
                         "the lower-triangle Q stream's); the other mode is measured too (one GPU) "
                         "and reported under 'other_mode'")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    from paper_2502_04640_b200 import xm
    from synth.scenes import CONFIG_DESCRIPTIONS, config_scene

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        nccl_id = share_id(dist, rank, xm.nccl_unique_id)

    sc = config_scene(args.config, seed=args.seed)
    dev = torch.device("cuda", local)
    d_fr = torch.from_numpy(sc.frame).to(dev)
    d_lm = torch.from_numpy(sc.landmark).to(dev)
    d_pts = torch.from_numpy(sc.pts).to(dev)
    d_w = torch.from_numpy(sc.w).to(dev)
    out_dev = dict(R=torch.empty((sc.N, 3, 3), dtype=torch.float64, device=dev),
                   s=torch.empty(sc.N, dtype=torch.float64, device=dev),
                   t=torch.empty((sc.N, 3), dtype=torch.float64, device=dev),
                   p=torch.empty((sc.M, 3), dtype=torch.float64, device=dev))
    stream = torch.cuda.current_stream(dev)
    implicit = 1 if args.mode == "implicit" else 0
    if args.mode == "auto":
        implicit = 1 if pick_implicit(sc.N, sc.E, world) else 0
    ctx = xm.Context(device=local, rank=rank, world=world, nccl_id=nccl_id,
                     stream=stream.cuda_stream, profile=0, implicit_q=implicit)

    def step(inputs, outputs):
        ctx.build_Q(sc.N, sc.M, *inputs)
        st, info = ctx.solve(3)
        cert = ctx.certify()
        ctx.round_recover_into(**outputs)
        return st, info, cert

    def barrier():
        if dist is not None:
            dist.barrier()

    dev_in = (d_fr, d_lm, d_pts, d_w)
    for _ in range(args.warmup):
        step(dev_in, out_dev)
    torch.cuda.synchronize()
    ctx.reset_stats()
    infos = []
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            infos.append(step(dev_in, out_dev))
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = max_over_ranks(dist, e0.elapsed_time(e1) / args.steps, dev)
    stats = ctx.stats()

    # ---- roofline pass: the same steps with CUDA events around every Q·V product
    aux_steps = min(args.steps, 5)          # roofline / e2e passes: at most 5 steps each
    pstats = roofline_pass(ctx, step, dev_in, out_dev, aux_steps, barrier)

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        h_in = tuple(torch.from_numpy(a).pin_memory() for a in (sc.frame, sc.landmark, sc.pts, sc.w))
        out_host = {k: torch.empty(v.shape, dtype=torch.float64).pin_memory() for k, v in out_dev.items()}
        step(h_in, out_host)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(aux_steps):
            step(h_in, out_host)
        torch.cuda.synchronize()
        barrier()
        e2e_s = max_over_ranks(dist, (time.perf_counter() - t0) / aux_steps, dev)
        e2e = {"value": e2e_s, "unit": "s", "steps": aux_steps,
               "h2d_bytes_per_step": int(sum(a.numel() * a.element_size() for a in h_in)),
               "d2h_bytes_per_step": int(sum(v.numel() * 8 for v in out_host.values()))}

    st, info, cert = infos[-1]
    value = ms / 1e3
    tkey = f"{args.config}_implicit" if implicit else args.config
    kname = KERNEL_IMPLICIT if implicit else (KERNEL_DENSE_B if sc.N < 4000 else KERNEL_DENSE)
    roof = roofline_obj(pstats, kname, traffic_of(tkey), ms, aux_steps)
    result = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config {args.config}: {CONFIG_DESCRIPTIONS[args.config]}",
                   "N": sc.N, "M": sc.M, "E": sc.E, "seed": args.seed,
                   "mode": "implicit (NEXT-1)" if implicit else "dense Q",
                   "parallelism": f"bands{world}",
                   "l2": ("inputs larger than L2 (per-measurement streams 0.4 GB + K̄⁻¹ lower triangle "
                          "0.41 GB per product > 126 MB)" if implicit else
                          "inputs larger than L2 (Q > 126 MB)")},
        "hvp_per_s": info["hvps"] / value if value > 0 else None,
        "solve": {"hvps": info["hvps"], "spmms": info["spmms"], "lanczos_steps": info["lanczos_steps"],
                  "outer_iters": info["outer_iters"], "r": info["r"], "escapes": info["escapes"],
                  "certified": info["certified"], "f": info["f"], "s_min": info["s_min"],
                  "lambda_min": cert["lambda_min"], "lambda_min_rel": cert["lambda_min"] / max(1.0, cert["normQ"]),
                  "lambda_lower": cert["lambda_lower"], "lower_rigorous": cert["lower_rigorous"],
                  "cert_method": ["lanczos(Z)", "cholesky(Z+eps*I) + shift-invert lanczos"][cert["method"]],
                  "eta": cert["eta"], "eta_rigorous": cert["eta_rigorous"],
                  "rho_hat": cert["rho_hat"], "status": st},
        "phases_ms": {k: stats[k] / args.steps for k in ("ms_build", "ms_solve", "ms_certify", "ms_round")},
        "roofline": roof,
        "gpu_launches": int(stats["kernel_launches"]),
        "e2e": e2e,
    }
    clocks = clk.summary()
    result["clocks"] = clocks
    if world == 1 and not args.no_other_mode:
        # the other product mode on the same workload (SURVEY §8(f) NEXT-1 vs the dense stream)
        other = 1 - implicit
        with xm.Context(device=local, stream=stream.cuda_stream, profile=0, implicit_q=other) as c2:
            def step2():
                c2.build_Q(sc.N, sc.M, *dev_in)
                st2, info2 = c2.solve(3)
                cert2 = c2.certify()
                c2.round_recover_into(**out_dev)
                return st2, info2, cert2
            for _ in range(2):
                step2()
            torch.cuda.synchronize()
            c2.reset_stats()
            o0 = torch.cuda.Event(enable_timing=True)
            o1 = torch.cuda.Event(enable_timing=True)
            o0.record(stream)
            k2 = min(args.steps, 5)
            for _ in range(k2):
                st2, info2, cert2 = step2()
            o1.record(stream)
            torch.cuda.synchronize()
            s2 = c2.stats()
            v2 = o0.elapsed_time(o1) / k2
            ps2 = roofline_pass(c2, lambda a, b: step2(), dev_in, out_dev, k2, lambda: None)
            roof2 = roofline_obj(ps2, KERNEL_IMPLICIT if other else (KERNEL_DENSE_B if sc.N < 4000
                                                                     else KERNEL_DENSE),
                                 traffic_of(f"{args.config}_implicit" if other else args.config), v2, k2)
            per_product = dense_bytes(sc.N, 3) if other == 0 else implicit_bytes(sc.N, sc.E, 3)
            result["other_mode"] = {
                "mode": "dense" if other == 0 else "implicit (NEXT-1, Q never formed)",
                "value": v2 / 1e3, "unit": "s", "steps": k2, "roofline": roof2,
                "phases_ms": {k: s2[k] / k2 for k in ("ms_build", "ms_solve", "ms_certify", "ms_round")},
                "hvps": info2["hvps"], "spmms": info2["spmms"], "r": info2["r"],
                "certified": info2["certified"], "eta": cert2["eta"], "status": st2,
                "alg_bytes_per_product": per_product}
    # the north star's "Q·Y SpMM at ≥ 60 % of HBM" metric: the dense lower-triangle
    # stream (k_spmm_sym), measured in this run in whichever mode ran it
    dense_roof = roof if not implicit else result.get("other_mode", {}).get("roofline")
    if dense_roof:
        result["spmm_roofline"] = {k: dense_roof[k] for k in
                                   ("kernel", "bound", "achieved", "peak", "unit", "frac", "traffic")}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        est = OracleEstimate(sc, args.config)
        if est.available():
            v, sample = est.step()
            result["cpu_baseline"] = {"value": v, "unit": "s", "cores": oracle_threads(),
                                      "kind": "oracle", "estimate": True, "cpu": cpu_model(),
                                      "sample": sample}
        else:
            result["cpu_baseline"] = None
    if rank == 0:
        print(json.dumps(result), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
