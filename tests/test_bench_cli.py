"""bench.py's launch contract, host side (no GPU): `--gpus N` without a
launcher starts N ranks (re-exec under torch.distributed.run on 127.0.0.1) and
the JSON line reports n_gpus == N; a WORLD_SIZE that disagrees with --gpus is
an error instead of a silent world-1 measurement."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=240):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                          env=e, capture_output=True, text=True, timeout=timeout)


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_gpus2_self_launches_two_ranks():
    r = _run(["--gpus", "2", "--dry-run", "--steps", "3"])
    assert r.returncode == 0, r.stdout + r.stderr
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["ranks_seen_max"] == 2.0
    assert d["windows_per_step"] == 2 * 256 * (10000 - 64 + 1)


def test_gpus3_c3_shards():
    r = _run(["--gpus", "3", "--dry-run", "--workload", "c3"])
    assert r.returncode == 0, r.stdout + r.stderr
    d = _line(r.stdout)
    assert d["n_gpus"] == 3 and d["config"]["parallelism"] == "instance-sharded x3"


def test_world_size_mismatch_is_an_error():
    r = _run(["--gpus", "4", "--dry-run"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=1" in r.stderr
