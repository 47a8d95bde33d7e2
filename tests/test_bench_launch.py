"""`python bench.py --gpus N` starts N ranks itself (the driver's plain launch), on CPU.

RSYLV_BENCH_DRYRUN=1 makes the re-exec'd torchrun ranks join a gloo group and report the world
size instead of running the solve, so the launcher is checked without a GPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                          capture_output=True, text=True, timeout=240)


def test_gpus_flag_starts_that_many_ranks():
    for n in (2, 3):
        p = _run(["--gpus", str(n), "--steps", "1", "--warmup", "3"], {"RSYLV_BENCH_DRYRUN": "1"})
        assert p.returncode == 0, p.stderr[-2000:]
        lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, p.stdout  # only rank 0 prints
        d = json.loads(lines[0])
        assert d["dry_run"] and d["n_gpus"] == n and d["ranks"] == n * (n - 1) // 2


def test_gpus_flag_fails_loudly_without_devices():
    import torch
    if torch.cuda.device_count() >= 2:
        return
    p = _run(["--gpus", "2"], {"RSYLV_BENCH_DRYRUN": "0"})
    assert p.returncode == 2 and "CUDA device" in p.stderr
