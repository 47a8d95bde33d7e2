"""Host-side logic of the multi-GPU path, on CPU: a 2-rank (and 3-rank) gloo group checks the
alpha reduction collectives, and the ownership / push-target rules are checked to deliver
every row-update source to exactly the ranks that consume it."""
import math
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1905_10574_b200 import dist as rdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for per_rank in cases:
            emin, numax = per_rank[rank]
            res.append(rdist.reduce_alpha(emin, numax, 8.98846567431158e307, dist))
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_alpha_reduction_over_gloo(world):
    cases = [
        [(0, 0.5), (0, 2.0), (0, 1.0)],                 # alpha = 1
        [(-10, 1e300), (-3, 1e307), (-20, 0.25)],       # norms re-based to the global minimum
        [(-5000, 1e300), (-4000, 8e307), (-4500, 0.0)],
    ]
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, cases, out), nprocs=world, join=True)
    for ci, per_rank in enumerate(cases):
        per = per_rank[:world]
        emin_g = min(e for e, _ in per)
        numax_g = max(math.ldexp(v, emin_g - e) if v > 0 else 0.0 for e, v in per)
        want = (rdist.alpha_exponent(emin_g, numax_g, 8.98846567431158e307), emin_g, numax_g)
        for r in range(world):
            got = out[r][ci]
            assert got[0] == want[0] and got[1] == want[1]
            assert got[2] == pytest.approx(want[2], rel=1e-15)


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("N", [1, 2, 5, 16, 79])
def test_push_targets_cover_exactly_the_consumers(R, N):
    for j in range(N):
        src_owner = rdist.owner(j, R)
        consumers = {rdist.owner(jp, R) for jp in range(j + 1, N)} - {src_owner}
        assert set(rdist.push_targets(j, N, R, src_owner)) == consumers


def test_alpha_exponent_matches_single_gpu_rule():
    om = 8.98846567431158e307
    assert rdist.alpha_exponent(0, 1.0, om) == 0
    assert rdist.alpha_exponent(-100, 1e300, om) == -100 + int(math.floor(math.log2(om / 1e300)))
    assert rdist.alpha_exponent(-100, 0.0, om) == 0
