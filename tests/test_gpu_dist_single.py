"""The multi-process path (paper_1905_10574_b200/dist.py: rsylv_b200_dist_prepare / _run /
_finish, CUDA-IPC handle exchange, NCCL alpha all-reduce) run end to end as a 1-rank NCCL job.

One rank owns every tile column, so nothing waits on another process (the pool gives one GPU per
call; ranks that wait on each other must not share a GPU). What this covers on the GPU: the
handle export/all-gather, the per-rank workspace and flag reset, the persistent kernel in its
distributed configuration, the NCCL MIN/MAX reduction of the exponent minima / tile norms and the
copy-out of the owned columns -- all of which bench.py --gpus N uses. The result must be
bitwise the single-process solve's. The exchange between ranks is covered by
tests/test_gpu_multirank.py (virtual ranks in one launch) and tests/test_dist_host.py (gloo).
"""
import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import sys
    import torch, torch.distributed as dist
    sys.path.insert(0, {root!r})
    from paper_1905_10574_b200 import api
    from paper_1905_10574_b200.configs import CONFIGS, device_system
    from paper_1905_10574_b200.dist import solve_dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    for name, m, n, t in {cases!r}:
        cfg = CONFIGS[name].scaled(m, n, t)
        A, ac, B, bc, C = device_system(cfg, torch)
        Yd = torch.full((cfg.n, cfg.m), float("nan"), dtype=torch.float64, device="cuda").T
        std, ae, rd = solve_dist(A, ac, B, bc, C, Yd, cfg.tile,
                                 stream=torch.cuda.current_stream().cuda_stream, device=0)
        torch.cuda.synchronize()
        Ys = torch.empty_like(Yd)
        sts, rs = api.solve_tiled_robust_device(A, ac, B, bc, C, Ys, cfg.tile, raise_underflow=False)
        torch.cuda.synchronize()
        same = torch.equal(Yd.view(torch.int64), Ys.view(torch.int64))
        print(name, m, n, t, "status", std, sts, "alpha_exp", ae, rs.alpha_exp, "bitwise", same,
              flush=True)
        assert std == sts and ae == rs.alpha_exp and same, name
    dist.destroy_process_group()
    print("DIST1 OK")
""")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_dist_path_one_rank_matches_single_process():
    cases = [("c1", 700, 500, 128), ("c5", 2048, 2048, 512), ("c3", 1536, 1536, 256),
             ("c4", 4096, 640, 256)]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, cases=cases)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "DIST1 OK" in p.stdout, p.stdout + p.stderr
