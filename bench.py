#!/usr/bin/env python3
"""Benchmark: FP64 GFLOP/s (m*n*(m+n)) of the robust triangular Sylvester solve on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl b200|reference]

One "step" = one full robust tiled solve (rsylv::solve_tiled_robust semantics: pack/bounds,
tile DAG, alpha reduction, consistency scaling) of BASELINE.json's largest configuration (c5:
m=n=40000, tile 512, 50% 2x2 blocks, 1% of C tiles x 1e250) with inputs resident in HBM.
Inputs are 12.8 GB per matrix, far larger than the 126 MB L2, so no L2 flush is needed.

* value  : whole-job GFLOP/s over the K timed steps (CUDA events on the solve stream,
           max over ranks).
* e2e    : the same metric through the reference-facing host API (rsylv_b200_solve) with pinned
           HOST buffers: H2D of A, B, C and D2H of Y inside the timed region.
* roofline: the tile-DAG kernel (DMMA update GEMMs + diagonal solves) against the measured
           FP64 DMMA peak of this pool's B200 (profiles/r01_fp64_peak_probe.log).
* cpu_baseline: the UNMODIFIED reference (oracle/_ref/librsylv_ref[_v4].so, built from
           /root/reference sources) on this host's cores: c1 at its literal size, the larger
           configs on a bounded sample, at the reference's best tile size.

--impl reference runs only the reference CPU path (rank 0) on that sample and prints its line.
Multi-GPU (N > 1): one process per GPU (torchrun); tile columns block-cyclic over the ranks, solved
tiles pushed to the consuming GPUs over NVLink (CUDA IPC), alpha via NCCL all-reduce MIN
(paper_1905_10574_b200/dist.py). The problem size is fixed: strong scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 37.05     # measured: tools/fp64_peak.cu on this pool's B200 (1965 MHz)
FP64_CUBLAS_TFLOPS = 35.46        # measured: cuBLAS DGEMM 8192^3 burst, same probe
CPU_SAMPLE = 1280                 # reference CPU sample edge (c5 distributions, tile 512)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c5")
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--scheduler", type=int, default=0)
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--force-dist", action="store_true",
                   help="run the multi-GPU path (dist.py, NCCL) even at N=1 (testing)")
    return p.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (200 ms period)."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def cpu_sample_cfg(cfg):
    """Bounded CPU sample of the workload. c1 (2000^2), the one config the reference solves, is
    run at its literal size (same_config). The others use the same distributions, hot tiles
    included, at CPU_SAMPLE^2: for c5 that is 1280^2 with one C tile x 1e250, which the
    reference completes WITH robust scaling (alpha = 3.3e-20), whereas the literal 40000^2
    system (and 1536^2, 2048^2 with this seed) ends in ScaleUnderflowError."""
    if cfg.m * cfg.n <= 2000 * 2000:
        return cfg
    s = min(CPU_SAMPLE, cfg.m, cfg.n)
    return cfg.scaled(s, s)


def run_cpu_reference(cfg, reps: int, seq: bool = False):
    """Times the unmodified reference rsylv::solve_tiled_robust (parallel mode, all host cores;
    the x86-64-v4 / AVX-512 build when the host has it, as the reference's -march=native build
    would) on the bounded sample, at the reference's best tile size among {128, 256, the
    config's}: its tile solve is super-cubic in the tile size, so the
    config's 512 would understate it. Returns the sample, the chosen tile, the step times
    at that tile and a description."""
    os.environ.setdefault("RSYLV_REF_VARIANT", "native")
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    from paper_1905_10574_b200.configs import host_system
    scfg = cpu_sample_cfg(cfg)
    a, ac, b, bc, c = host_system(scfg)
    cores = os.cpu_count() or 1
    per_tile = {}
    for t in sorted({128, 256, scfg.tile}):
        t0 = time.perf_counter()
        r = po.solve_tiled(a, ac, b, bc, c, t, impl="ref", workers=cores)
        per_tile[t] = (time.perf_counter() - t0, r.status)
    best = min(per_tile, key=lambda t: per_tile[t][0])
    times, status = [], per_tile[best][1]
    for _ in range(max(0, reps - 1)):
        t0 = time.perf_counter()
        r = po.solve_tiled(a, ac, b, bc, c, best, impl="ref", workers=cores)
        times.append(time.perf_counter() - t0)
        status = r.status
    times = [per_tile[best][0]] + times
    extra = {"tiles_s": {str(t): round(v[0], 4) for t, v in per_tile.items()},
             "build": f"x86-64-{po.ref_variant()}", "same_config": scfg is cfg}
    if seq:
        t0 = time.perf_counter()
        po.solve_tiled(a, ac, b, bc, c, best, impl="ref", workers=0)
        extra["sequential_s"] = round(time.perf_counter() - t0, 4)
        extra["sequential_gflops"] = scfg.flops() / extra["sequential_s"] / 1e9
    sample = (f"reference rsylv::solve_tiled_robust, parallel({cores}), {scfg.m}x{scfg.n} at its "
              f"best tile {best} (of {sorted(per_tile)}), {cfg.name} distributions (hot tiles "
              f"included), {extra['build']} build; status {po.STATUS_NAMES[status]}")
    return scfg, best, times, cores, sample, extra


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    from paper_1905_10574_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if rank != 0:
        return
    scfg, best, times, cores, sample, extra = run_cpu_reference(
        cfg, args.warmup + args.steps, seq=scfg_is_small(cfg))
    timed = times[args.warmup:] or times
    t = sum(timed)
    val = scfg.flops() * len(timed) / t / 1e9
    line = {"impl": "reference", "metric": "FP64 GFLOP/s (m*n*(m+n)) robust Sylvester solve",
            "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": len(timed),
            "warmup": args.warmup, "ms_per_step": 1e3 * t / len(timed), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.note}", "sample": f"{scfg.m}x{scfg.n}",
                       "tile": best, "config_tile": cfg.tile,
                       "same_config": extra["same_config"]},
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cores,
                             "kind": "reference", "sample": sample, **extra},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def scfg_is_small(cfg) -> bool:
    """Configs the reference completes at their literal size in seconds (c1): also timed in
    sequential() mode."""
    return cfg.m * cfg.n <= 2000 * 2000


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_relaunch(args) -> None:
    """`python bench.py --gpus N` with N > 1 outside torchrun: re-exec this script under
    torch.distributed.run with N processes (one per GPU), so that the number of GPUs measured is
    the number asked for. Fails loudly when fewer than N devices are visible (never silently
    measures fewer). RSYLV_BENCH_DRYRUN=1 runs the same launch on CPU with gloo ranks that only
    report the world size (tests/test_bench_launch.py)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    dry = os.environ.get("RSYLV_BENCH_DRYRUN") == "1"
    if not dry:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) "
                             "are visible\n")
            sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dry_run(args) -> None:
    """RSYLV_BENCH_DRYRUN=1 under torchrun: a gloo all-reduce over the ranks the launcher
    started; rank 0 prints {"dry_run": true, "n_gpus": world, "ranks": sum of ranks}."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    world, rank = dist.get_world_size(), dist.get_rank()
    t = torch.tensor([rank], dtype=torch.int64)
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "gpus_arg": args.gpus,
                          "ranks": int(t.item())}), flush=True)
    dist.destroy_process_group()


def group_e2e(args, cfg, ocfg, A, ac, B, bc, Cm, rank, world):
    """e2e at N > 1: rank 0 solves through the reference-facing multi-GPU host entry
    (rsylv_b200_solve_group over GPUs 0 .. N-1 of this node: what ExecutionMode::parallel(N)
    reaches through the shim) with pinned HOST buffers; H2D of A, B (upper tiles, to every GPU)
    and of each GPU's C columns, D2H of Y inside the timed region. The other ranks free their
    device tensors and wait on the rendezvous store (no GPU work meanwhile)."""
    import torch
    import torch.distributed as dist
    import ctypes as C
    from paper_1905_10574_b200 import _native as nat
    store = dist.distributed_c10d._get_default_store()
    out = None
    if rank == 0:
        try:
            hA = torch.empty((cfg.m, cfg.m), dtype=torch.float64, pin_memory=True)
            hB = torch.empty((cfg.n, cfg.n), dtype=torch.float64, pin_memory=True)
            hC = torch.empty((cfg.n, cfg.m), dtype=torch.float64, pin_memory=True)
            hY = torch.empty((cfg.n, cfg.m), dtype=torch.float64, pin_memory=True)
            hA.copy_(A.T)
            hB.copy_(B.T)
            hC.copy_(Cm.T)
            torch.cuda.synchronize()
            L = nat.lib()
            opt = nat.Options(ocfg.omega, ocfg.small_num, cfg.tile, 0, 0)
            ctxs = (C.c_void_p * world)(*[nat.context(d) for d in range(world)])
            up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))  # noqa: E731
            dp = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_double))  # noqa: E731
            times = []
            for it in range(args.e2e_steps + 1):
                r = nat.Result()
                t0 = time.perf_counter()
                st = L.rsylv_b200_solve_group(ctxs, world, cfg.m, cfg.n, dp(hA), cfg.m, up(ac),
                                              dp(hB), cfg.n, up(bc), dp(hC), cfg.m, dp(hY),
                                              cfg.m, C.byref(opt), C.byref(r))
                dt = time.perf_counter() - t0
                if st not in (nat.RSYLV_OK, nat.RSYLV_SCALE_UNDERFLOW):
                    raise RuntimeError(f"rsylv_b200_solve_group: status {st}")
                if it > 0:
                    times.append(dt)
            tmean = sum(times) / len(times)
            out = {"value": cfg.flops() / tmean / 1e9, "unit": "GFLOP/s",
                   "h2d_bytes_per_step": int(r.h2d_bytes), "d2h_bytes_per_step": int(r.d2h_bytes),
                   "ms_per_step": 1e3 * tmean,
                   "api": f"rsylv_b200_solve_group over {world} GPUs (host buffers, pinned)"}
            del hA, hB, hC, hY
        except Exception as e:  # never lose the device-resident line
            sys.stderr.write(f"bench.py: group e2e failed: {e}\n")
            out = None
        store.set("rsylv_e2e_done", "1")
    else:
        torch.cuda.synchronize()
        store.wait(["rsylv_e2e_done"])
    return out


def main():
    args = parse()
    maybe_relaunch(args)
    if os.environ.get("RSYLV_BENCH_DRYRUN") == "1":
        dry_run(args)
        return
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != max(1, args.gpus):
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    use_dist = world > 1 or args.force_dist  # --force-dist: the multi-GPU path at any N
    torch.cuda.set_device(local)
    json_out = sys.stdout
    if use_dist:
        # NCCL writes its banner ("NCCL version ...") to fd 1 when NCCL_DEBUG asks for it; keep
        # stdout for the one JSON line and send everything else to stderr
        sys.stdout.flush()
        json_out = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1905_10574_b200 import api, _native as nat
    from paper_1905_10574_b200.configs import CONFIGS, device_system
    cfg = CONFIGS[args.config]
    stream = torch.cuda.current_stream()
    A, ac, B, bc, Cm = device_system(cfg, torch)
    Y = torch.empty((cfg.n, cfg.m), dtype=torch.float64, device="cuda").T
    ocfg = api.OverflowConfig()

    def step():
        if use_dist:
            from paper_1905_10574_b200.dist import solve_dist
            st, _, res = solve_dist(A, ac, B, bc, Cm, Y, cfg.tile, ocfg, stream=stream.cuda_stream,
                                    device=local)
            return st, res
        st, res = api.solve_tiled_robust_device(A, ac, B, bc, Cm, Y, cfg.tile, ocfg,
                                                stream=stream.cuda_stream,
                                                scheduler=args.scheduler, device=local,
                                                raise_underflow=False)
        return st, res

    for _ in range(args.warmup):
        st, res = step()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dag_ms, statuses = [], []
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            st, res = step()
            dag_ms.append(res.dag_ms)
            statuses.append(st)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if use_dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    torch.cuda.synchronize()
    ms_step = ms / args.steps
    value = cfg.flops() / (ms_step / 1e3) / 1e9  # one solve per step, split over the ranks
    if use_dist:  # every owned tile column (the solver's own partition)
        cuts = api.tile_cuts(bc, cfg.n, cfg.tile)
        finite = all(bool(torch.isfinite(Y[:, cuts[j]:cuts[j + 1]]).all().item())
                     for j in range(len(cuts) - 1) if j % world == rank)
    else:
        finite = bool(torch.isfinite(Y).all().item())
    alpha_exp = int(res.alpha_exp)

    # e2e through the host API with pinned buffers
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0 and not use_dist:
        # pinned host copies holding the column-major matrices (the storage of the .T views)
        hA = torch.empty((cfg.m, cfg.m), dtype=torch.float64, pin_memory=True)
        hB = torch.empty((cfg.n, cfg.n), dtype=torch.float64, pin_memory=True)
        hC = torch.empty((cfg.n, cfg.m), dtype=torch.float64, pin_memory=True)
        hY = torch.empty((cfg.n, cfg.m), dtype=torch.float64, pin_memory=True)
        hA.copy_(A.T)
        hB.copy_(B.T)
        hC.copy_(Cm.T)
        torch.cuda.synchronize()
        import ctypes as C
        L = nat.lib()
        opt = nat.Options(ocfg.omega, ocfg.small_num, cfg.tile, args.scheduler, 0)
        ctx = nat.context(local)
        up = lambda x: x.ctypes.data_as(C.POINTER(C.c_ubyte))  # noqa: E731
        dp = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_double))  # noqa: E731
        times = []
        for it in range(args.e2e_steps + 1):
            r = nat.Result()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s = L.rsylv_b200_solve(ctx, cfg.m, cfg.n, dp(hA), cfg.m, up(ac), dp(hB), cfg.n, up(bc),
                                   dp(hC), cfg.m, dp(hY), cfg.m, C.byref(opt), C.byref(r))
            dt = time.perf_counter() - t0
            if it > 0:  # first call warms the host-path staging buffers
                times.append(dt)
        if use_dist:
            t = torch.tensor([max(times)], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tmax = float(t.item())
        else:
            tmax = sum(times) / len(times)
        e2e = {"value": cfg.flops() * world / tmax / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(r.h2d_bytes),
               "d2h_bytes_per_step": int(r.d2h_bytes),
               "ms_per_step": 1e3 * tmax, "api": "rsylv_b200_solve (host buffers, pinned)"}
        del hA, hB, hC, hY

    if not args.no_e2e and args.e2e_steps > 0 and use_dist and world > 1:
        e2e = group_e2e(args, cfg, ocfg, A, ac, B, bc, Cm, rank, world)
        del A, B, Cm, Y

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        scfg, best, times, cores, sample, extra = run_cpu_reference(cfg, 1, seq=scfg_is_small(cfg))
        cpu = {"value": scfg.flops() / times[0] / 1e9, "unit": "GFLOP/s", "cores": cores,
               "kind": "reference", "sample": sample, **extra}

    # DRAM traffic of the dominant kernel per launch, from the committed ncu capture of the same
    # command (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k k_persistent)
    traffic, traffic_src = None, None
    here = os.path.dirname(os.path.abspath(__file__))
    tpath = next((p for p in (os.path.join(here, "profiles", r, f"traffic_{cfg.name}_k_persistent.csv")
                              for r in ("r02", "r01")) if os.path.exists(p)), "")
    if os.path.exists(tpath) and args.scheduler == 0 and world == 1:
        import csv
        vals = {}
        with open(tpath) as fh:
            for r in csv.reader(l for l in fh if not l.startswith("==")):
                if len(r) > 14 and r[12].startswith("dram__bytes"):
                    vals[r[12]] = float(r[14].replace(",", ""))
        if len(vals) == 2:
            traffic = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
            traffic_src = os.path.relpath(tpath, os.path.dirname(os.path.abspath(__file__)))

    dag = sum(dag_ms) / len(dag_ms)
    achieved = cfg.flops() / (dag / 1e3) / 1e12
    if rank == 0:
        line = {
            "metric": "FP64 GFLOP/s (m*n*(m+n)) robust Sylvester solve",
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.note}", "m": cfg.m, "n": cfg.n,
                       "tile": cfg.tile, "internal_tile": min(cfg.tile, api.INTERNAL_TILE),
                       "scheduler": "persistent" if args.scheduler == 0
                       else "wavefront", "l2": "inputs 12.8 GB/matrix >> 126 MB L2, no flush",
                       "parallelism": (f"tile columns block-cyclic over {world} GPUs, NVLink "
                                       "tile push + NCCL alpha all-reduce") if use_dist else "1 GPU",
                       "alpha_exp": alpha_exp, "status": nat.lib().rsylv_b200_status_string(
                           statuses[-1]).decode(), "y_finite": finite,
                       "scaling_events": int(res.scaling_events)},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_DMMA_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved / FP64_DMMA_PEAK_TFLOPS,
                         "traffic": traffic, "traffic_unit": "bytes per launch (DRAM read+write)",
                         "traffic_source": traffic_src,
                         "algorithmic_bytes": cfg.alg_bytes() if hasattr(cfg, "alg_bytes") else None,
                         "kernel": "k_persistent (tile DAG)",
                         "peak_source": "measured FP64 DMMA microbenchmark (profiles/"
                                        "r01_fp64_peak_probe.log); cuBLAS DGEMM 35.46"},
            "clocks": clk.summary(),
            "e2e": e2e,
            "e2e_note": None if e2e else ("group e2e failed (see stderr)" if use_dist and world > 1
                                          and not args.no_e2e else "disabled (--no-e2e)"),
            "cpu_baseline": cpu,
            "gpu_launches": args.steps * (4 + int(res.dag_launches)),
            "breakdown_ms": {"pack": res.pack_ms, "dag": dag, "unpack": res.unpack_ms},
        }
        print(json.dumps(line), file=json_out, flush=True)
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
