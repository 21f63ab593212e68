"""N > 1 host logic on CPU: world_size-2 gloo runs under torchrun (127.0.0.1).

* tests/_gloo_worker.py — id broadcast, max-over-ranks timing, row sharding and
  the padded all-gather layout (xm_shard_rows), ‖Q‖² all-reduce;
* bench.py --impl reference under torchrun — rank 0 alone prints one JSON line,
  the other rank exits 0 without work.
"""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun(args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}"] + args
    env = dict(os.environ, OMP_NUM_THREADS="1", CUDA_VISIBLE_DEVICES="")
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_gloo_sharding_and_plumbing():
    p = torchrun([os.path.join(ROOT, "tests", "_gloo_worker.py")])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "GLOO_OK" in p.stdout


def test_reference_arm_under_torchrun():
    p = torchrun(["bench.py", "--impl", "reference", "--gpus", "2", "--config", "A",
                  "--steps", "1", "--warmup", "3"])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
