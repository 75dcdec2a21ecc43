#!/usr/bin/env python3
"""bench.py -- vertices/s through OI track + project + reconstruct (BASELINE.json).

Default workload: config 5 (64 independent 512x512 grid meshes, 128 tiles of
32x64 = 2048 vertices each, c = 200, one warm-started OI step per tile, fp64),
the batched configuration the metric's multi-GPU scaling is quoted on.  One
"step" = every mesh of the job carried through the full chain: Laplacian
assembly, factorisation, first-submesh basis, OI tracking, projection, stitched
reconstruction (+ the NCCL gather of per-mesh results to all ranks when N > 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5|C2|C3|C4]
  python bench.py --impl reference ...     # CPU oracle (port) arm

Chains shard across ranks with no data-path collective.  Default: weak
scaling -- each GPU carries config 5's 64-mesh shard (mesh ids rank*64 ..
rank*64+63, each its own seed), the job grows with N; `--strong` splits the 64
meshes over the N GPUs instead.  The per-mesh reconstructions are all-gathered
(NCCL over NVLink) at the end of every step.  Timing: W untimed warm-up steps, then K steps
bracketed by barrier + synchronize, CUDA events on the launching device, max
over ranks.  Inputs (0.9 GB for C5) exceed the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "vertices/sec through OI track+project+reconstruct; % of HBM/FP64 roofline"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_TFLOPS = 37.18  # DMMA mma.sync f64, profiles/fp64_peak_r01.txt (measured on this pool's B200)

CONFIGS = {
    # name: (W, H, tile_w, tile_h, c, t, meshes, sigma, seed0)
    "C5": dict(W=512, H=512, tw=64, th=32, c=200, t=1, meshes=64, sigma=0.01, seed0=5000,
               desc="64 x 512^2 grid meshes, 128 tiles of 32x64 (n_d=2048) each, c=200, t=1"),
    # F3: denoise_dynamic of a frame sequence on config 5's grid and tiles
    "F3": dict(W=512, H=512, tw=64, th=32, c=200, t=1, meshes=1, frames=64, sigma=0.01, seed0=7000,
               desc="denoise_dynamic: 64 frames of a 512^2 grid sequence, 128 tiles of 32x64 (n_d=2048), "
                    "bases from frame 0 (c=200, t=1), every frame projected + stitched"),
    # F4: fine_denoise of config 4's 1024^2 noisy grid (2 M faces)
    "F4": dict(W=1024, H=1024, tw=64, th=64, c=0, t=0, meshes=1, fine=True, sigma=0.01, seed0=404,
               desc="fine_denoise (bilateral normals x5 over 1-rings + 10 vertex passes) of the 1024^2 noisy grid "
                    "(1 048 576 vertices, 2 093 058 faces), reference default BilateralParams"),
    "C2": dict(W=256, H=256, tw=32, th=32, c=100, t=1, meshes=1, sigma=0.005, seed0=202,
               desc="256^2 grid, 64 tiles of 32x32 (n_d=1024), c=100, t=1"),
}
PINNED = dict(weighting="binary", power=2, shift_scale=1e-3, dense_limit=4096)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--meshes", type=int, default=0, help="override the per-GPU mesh count (debug)")
    ap.add_argument("--strong", action="store_true", help="split the config's meshes over the GPUs (strong scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tiles", type=int, default=8, help="tiles per chain in the CPU sample")
    return ap.parse_args()


# ----------------------------------------------------------------------- inputs

def build_inputs(cfg, mesh_ids):
    import numpy as np
    from paper_1810_02719_b200 import synth
    base = synth.grid_mesh(cfg["W"], cfg["H"], cfg["seed0"], cfg["sigma"])
    seg = synth.grid_tiles(cfg["W"], cfg["H"], cfg["tw"], cfg["th"])
    verts = [synth.grid_vertices(cfg["W"], cfg["H"], cfg["seed0"] + i, cfg["sigma"]) for i in mesh_ids]
    offs, members = seg.flat()
    return base, seg, verts, np.asarray(offs, np.int32), np.asarray(members, np.int32)


# ----------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------- GPU arm

class GpuJob:
    def __init__(self, cfg, mesh_ids, device, ctx):
        import numpy as np
        import torch
        from paper_1810_02719_b200 import _abi
        self.cfg, self.ids, self.ctx, self.np = cfg, mesh_ids, ctx, np
        base, seg, verts, offs, members = build_inputs(cfg, mesh_ids)
        self.seg = seg
        self.n = base.n
        self.K = seg.count
        self.nd = seg.block_size
        self.B = len(mesh_ids)
        c = cfg["c"]
        dev = torch.device("cuda", device)
        self.torch, self.dev = torch, dev
        seq = np.arange(self.K, dtype=np.int32)
        # device-resident inputs (value) and pinned host inputs (e2e)
        self.d_xyz = [[torch.from_numpy(np.ascontiguousarray(v[:, a])).to(dev) for a in range(3)] for v in verts]
        self.h_xyz = [[torch.from_numpy(np.ascontiguousarray(v[:, a])).pin_memory() for a in range(3)] for v in verts]
        conn = dict(offs=base.adj_offsets, cols=base.adj_cols, moffs=offs, members=members, seq=seq)
        self.d_conn = {k: torch.from_numpy(np.asarray(a, np.int32)).to(dev) for k, a in conn.items()}
        self.h_conn = {k: torch.from_numpy(np.asarray(a, np.int32)).pin_memory() for k, a in conn.items()}
        # outputs
        self.ncoef = self.K * c * 3
        self.d_recon = torch.empty((self.B, 3 * self.n), dtype=torch.float64, device=dev)
        self.d_coef = torch.empty((self.B, self.ncoef), dtype=torch.float64, device=dev)
        self.h_recon = torch.empty((self.B, 3 * self.n), dtype=torch.float64).pin_memory()
        self.h_coef = torch.empty((self.B, self.ncoef), dtype=torch.float64).pin_memory()
        self.stats = [np.zeros((5, self.K)) for _ in range(self.B)]
        self.coef_off = [np.zeros(self.K + 1, np.int64) for _ in range(self.B)]
        self.sizes = np.full(self.K, c, np.int32)
        self.pcfg = _abi.smg_pipeline_config()
        ctx.lib.smg_default_config(self.pcfg)
        self.pcfg.weighting = _abi.WEIGHTING[PINNED["weighting"]]
        self.pcfg.subspace_size = c
        self.pcfg.iterations = cfg["t"]
        self.pcfg.power = PINNED["power"]
        self.pcfg.shift_scale = PINNED["shift_scale"]
        self._abi = _abi
        self.views = {on: self._views(on) for on in (0, 1)}
        # per-mesh coordinates + the shared topology once (the library stages host
        # arrays that several chains pass by the same pointer only once)
        self.h2d_bytes = sum(t.numel() * t.element_size() for xyz in self.h_xyz for t in xyz) + sum(
            self.h_conn[k].numel() * self.h_conn[k].element_size() for k in ("offs", "cols", "members"))
        self.d2h_bytes = self.h_recon.numel() * 8 + self.h_coef.numel() * 8 + self.B * 5 * self.K * 8

    def _views(self, on_device):
        _abi, np = self._abi, self.np
        xyz = self.d_xyz if on_device else self.h_xyz
        conn = self.d_conn if on_device else self.h_conn
        recon = self.d_recon if on_device else self.h_recon
        coef = self.d_coef if on_device else self.h_coef
        meshes = (_abi.smg_mesh * self.B)()
        segs = (_abi.smg_segmentation * self.B)()
        outs = (_abi.smg_chain_output * self.B)()
        for b in range(self.B):
            m = meshes[b]
            m.vertex_count = self.n
            m.x, m.y, m.z = (t.data_ptr() for t in xyz[b])
            m.adj_offsets, m.adj_cols = conn["offs"].data_ptr(), conn["cols"].data_ptr()
            m.on_device = on_device
            s = segs[b]
            s.submesh_count, s.member_offsets, s.members = self.K, conn["moffs"].data_ptr(), conn["members"].data_ptr()
            s.sequence_length, s.sequence, s.on_device = self.K, conn["seq"].data_ptr(), on_device
            o = outs[b]
            st = self.stats[b]
            o.subspace_size = None
            o.residual_rms = st[1].ctypes.data
            o.doi_residual = st[2].ctypes.data
            o.converged = None
            o.oi_iterations = None
            o.reconstruction = recon[b].data_ptr()
            o.coefficients = coef[b].data_ptr()
            o.coefficients_capacity = self.ncoef
            o.coefficient_offsets = self.coef_off[b].ctypes.data
            o.on_device = on_device
        return meshes, segs, outs

    def run(self, on_device):
        meshes, segs, outs = self.views[on_device]
        st = self.ctx.lib.smg_run_chains(self.ctx.handle, self.B, meshes, segs, self.pcfg,
                                         self.sizes.ctypes.data, outs)
        self.ctx.check(st)


def gpu_arm(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch
    import paper_1810_02719_b200 as G
    from paper_1810_02719_b200 import shard
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    per_gpu = args.meshes or cfg["meshes"]
    total_meshes = per_gpu if args.strong else per_gpu * world
    if cfg["meshes"] == 1:  # single-chain configs: replicas only
        ids = [rank]
        total_units = world
    else:
        ids = shard.shard_meshes(total_meshes, world, rank)
        total_units = total_meshes
    ctx = G.Context(local_rank)
    job = GpuJob(cfg, ids, local_rank, ctx)
    verts_per_unit = job.n
    gather = dist is not None and cfg["meshes"] > 1

    def step(on_device):
        job.run(on_device)
        if gather and on_device:
            # per-mesh reconstructions to every rank (NCCL over NVLink)
            shard.gather_meshes(job.d_recon, total_meshes)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(on_device, steps, profile=False):
        lib = ctx.lib
        if profile:
            lib.smg_profile_enable(ctx.handle, 1)
        l0 = launches()
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(steps):
            step(on_device)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        barrier()
        nl = launches() - l0
        if dist is not None:
            t = torch.tensor([ms], dtype=torch.float64, device=job.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, nl

    def launches():
        import ctypes as C
        n, t = C.c_int64(), C.c_double()
        ctx.lib.smg_profile_read(ctx.handle, b"launches", C.byref(n), C.byref(t))
        return n.value

    for _ in range(args.warmup):
        step(True)
    with ClockSampler(local_rank) as clk:
        ms, nl = timed(True, args.steps, profile=True)
    clocks = clk.summary()
    stages = {}
    import ctypes as C
    for nm in ("assemble", "factor", "first_basis", "fb_iterate", "fb_filter", "fb_rayleigh_ritz", "solve", "orthonormalize",
               "gram", "chol", "trmm", "project"):
        n, t = C.c_int64(), C.c_double()
        ctx.lib.smg_profile_read(ctx.handle, nm.encode(), C.byref(n), C.byref(t))
        stages[nm] = {"launches": n.value, "ms": t.value / args.steps}
    ctx.lib.smg_profile_enable(ctx.handle, 0)
    # e2e: host pinned inputs -> results on the host
    step(False)
    ms_e2e, _ = timed(False, args.steps)

    ms_step = ms / args.steps
    units = total_units * verts_per_unit
    value = units / (ms_step / 1e3)
    e2e_value = units / (ms_e2e / args.steps / 1e3)

    # roofline of the dominant kernel (solve: the block-tridiagonal R^z sweeps).
    # Algorithmic flops: z*4*n_d*b*c per tile and OI iteration,
    # b = half-bandwidth in the natural order; the "solve" stage also holds the
    # first basis's shift-invert bootstrap (4 iterations on m columns, the first
    # with z = 1).  Launch durations are CUDA-event spans on the launching
    # stream inside the timed region; two chain groups share the GPU, so a
    # launch's span includes time the other group's kernels occupy SMs.
    c, n, B, K, t = cfg["c"], job.nd, job.B, job.K, cfg["t"]
    b_half = cfg["tw"] + 1
    z = PINNED["power"]
    m_fb = min(n, max(c, min(480, -(-(c + max(16, c // 2)) // 8) * 8)))
    solve = stages["solve"]
    solve_launches_per_step = solve["launches"] / args.steps if solve["launches"] else 0
    solve_flops_step = B * ((K - 1) * t * z * 4.0 * n * b_half * c + (1 + 3 * z) * 4.0 * n * b_half * m_fb)
    flops_per_launch = solve_flops_step / max(solve_launches_per_step, 1e-9)
    avg_ms = solve["ms"] / max(solve_launches_per_step, 1e-9)
    achieved = solve_flops_step / (solve["ms"] * 1e-3) / 1e12 if solve["ms"] > 0 else None
    traffic = None
    try:  # dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "solve_traffic_r01.json")) as f:
            traffic = json.load(f)["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        pass
    # the factorisation's ordering picks the block width: the geometric order gives
    # 32x64 grid tiles W = 32 (band 33) where the natural order has 65, so the
    # DMMA work done is below the SURVEY's algorithmic figure (kept as the
    # contract's numerator); hw_flops_per_launch is the block solve's own count
    W_used = 32 if B * K >= 2048 else 64
    # per triangular sweep 3*n*W*cols flops (triangular half + full coupling half);
    # an OI step is 2z sweeps, the bootstrap 2 + 3*2z sweeps on m columns
    hw_step = B * 3.0 * n * W_used * ((K - 1) * t * 2 * z * c + (2 + 3 * 2 * z) * m_fb)
    roofline = {"kernel": "solve_kernel (block-tridiagonal R^z sweeps, DMMA f64)", "bound": "tensor",
                "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None, "traffic": traffic,
                "traffic_source": "profiles/solve_traffic_r01.json (bytes per launch of 32 chains)",
                "peak_source": "measured FP64 DMMA peak, profiles/fp64_peak_r01.txt (MEASURED_PEAKS.json has no FP64 entry)",
                "flops_per_launch": flops_per_launch, "avg_launch_ms": avg_ms,
                "b_algorithmic": b_half, "block_width_used": W_used,
                "hw_flops_per_launch": hw_step / max(solve_launches_per_step, 1e-9),
                "hw_frac": (hw_step / (solve["ms"] * 1e-3) / 1e12 / FP64_PEAK_TFLOPS) if solve["ms"] > 0 else None,
                "launches_per_step": solve_launches_per_step,
                "step_share": solve["ms"] / ms_step if ms_step else None}
    # whole-step algorithmic FP64 work (SURVEY.md §8(d) formulas, per GPU)
    per_tile = z * 4.0 * n * b_half * c * t + (4.0 * n * c * c) * t + n * b_half ** 2 + 12.0 * n * c + 3 * n
    first = (4.0 / 3.0) * n ** 3 + 2.0 * n * n * c
    step_flops = B * ((K - 1) * per_tile + first)
    out = {
        "metric": METRIC, "value": value, "unit": "vertices/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong" if (args.strong and cfg["meshes"] > 1) else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded sinusoid height-field grids + N(0,sigma^2) noise; no dataset exists)",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "meshes": total_units, "meshes_per_gpu": len(ids),
                   "tiles_per_mesh": K,
                   "n_d": n, "c": c, "oi_iterations": t, "z": z, "shift_scale": PINNED["shift_scale"],
                   "weighting": PINNED["weighting"], "tile_order": "row-major",
                   "parallelism": (f"chains sharded over {world} GPU(s), "
                                   + (f"{total_meshes} meshes split (strong)" if args.strong
                                      else f"{len(ids)} meshes per GPU (weak)")) if cfg["meshes"] > 1 else "replicas",
                   "l2": "inputs larger than L2 (%.0f MB per GPU)" % (job.h2d_bytes / 1e6)},
        "e2e": {"value": e2e_value, "unit": "vertices/s", "h2d_bytes_per_step": job.h2d_bytes,
                "d2h_bytes_per_step": job.d2h_bytes},
        "roofline": roofline,
        "fp64_step_efficiency": {"algorithmic_tflop_per_step": step_flops / 1e12,
                                 "achieved_tflops": step_flops / (ms_step * 1e-3) / 1e12,
                                 "frac_of_peak": step_flops / (ms_step * 1e-3) / 1e12 / FP64_PEAK_TFLOPS},
        "stages_ms_per_step": {k: round(v["ms"], 3) for k, v in stages.items()},
        "clocks": clocks,
        "gpu_launches": nl,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, cfg, total_units)
    if dist is not None:
        dist.destroy_process_group()
    ctx.close()
    return out if rank == 0 else None


# ----------------------------------------------------------------------- CPU arm

def _cpu_chain(task):
    """One chain of the oracle over the first T tiles: (t_first, t_rest) seconds."""
    cfgname, mesh_id, T = task
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import specmesh_oracle as O
    from paper_1810_02719_b200 import synth
    cfg = CONFIGS[cfgname]
    base = synth.grid_mesh(cfg["W"], cfg["H"], cfg["seed0"] + mesh_id, cfg["sigma"])
    seg = synth.grid_tiles(cfg["W"], cfg["H"], cfg["tw"], cfg["th"])
    subs = O.build_submeshes(base.adj_offsets, base.adj_cols, seg.members[:T])
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=cfg["c"], iterations=cfg["t"],
                            shift_scale=PINNED["shift_scale"])
    t0 = time.perf_counter()
    bb1 = O.compute_block_bases_fixed_sizes(base.vertices, subs[:1], np.arange(1), ocfg, [cfg["c"]])
    O.project_blocks(bb1, base.vertices)
    t1 = time.perf_counter()
    bb = O.compute_block_bases_fixed_sizes(base.vertices, subs, np.arange(T), ocfg, [cfg["c"]] * T)
    locals_ = O.project_blocks(bb, base.vertices)
    t2 = time.perf_counter()
    return t1 - t0, (t2 - t1) - (t1 - t0)


def cpu_baseline(args, cfg, total_units):
    """The oracle restatement timed on the host cores (one chain per core, BLAS 1 thread),
    on a bounded sample: the first T tiles of P chains, extrapolated per chain to all tiles."""
    import multiprocessing as mp
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["MKL_NUM_THREADS"] = "1"
    cores = os.cpu_count() or 1
    P = min(cores, max(1, total_units if cfg["meshes"] > 1 else 1))
    T = max(2, args.cpu_tiles)
    K = (cfg["W"] // cfg["tw"]) * (cfg["H"] // cfg["th"])
    T = min(T, K)
    ctxm = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctxm.Pool(P) as pool:
        res = pool.map(_cpu_chain, [(args.config, i, T) for i in range(P)])
    wall = time.perf_counter() - t0
    t_first = sum(r[0] for r in res) / P
    t_rest = sum(r[1] for r in res) / P / max(T - 1, 1)
    t_chain = t_first + (K - 1) * t_rest
    n_mesh = cfg["W"] * cfg["H"]
    rounds = math.ceil(total_units / P)
    value = total_units * n_mesh / (rounds * t_chain)
    return {"value": value, "unit": "vertices/s", "cores": P, "kind": "port",
            "sample": f"{P} chains in parallel (1 per core, BLAS 1 thread) x first {T} of {K} tiles "
                      f"(numpy/LAPACK oracle, oracle/specmesh_oracle.py); per chain t_first={t_first:.2f}s "
                      f"+ {K - 1} x t_tile={t_rest:.3f}s extrapolated; sample wall {wall:.1f}s"}


def reference_arm(args, cfg):
    total_units = (args.meshes or cfg["meshes"]) * (1 if args.strong else max(1, args.gpus))
    vals = []
    for _ in range(max(1, args.steps)):
        cb = cpu_baseline(args, cfg, total_units)
        vals.append(cb["value"])
    cb["value"] = statistics.median(vals)
    n_mesh = cfg["W"] * cfg["H"]
    ms_step = total_units * n_mesh / cb["value"] * 1e3
    return {"metric": METRIC, "value": cb["value"], "unit": "vertices/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if (args.strong and cfg["meshes"] > 1) else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded sinusoid height-field grids + N(0,sigma^2) noise)",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "meshes": total_units},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "vertices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ----------------------------------------------------------------------- F3 arm

def _frames_inputs(cfg, seed):
    from paper_1810_02719_b200 import synth
    topo = synth.grid_mesh(cfg["W"], cfg["H"], seed, cfg["sigma"])
    seg = synth.grid_tiles(cfg["W"], cfg["H"], cfg["tw"], cfg["th"])
    verts = synth.grid_sequence(cfg["W"], cfg["H"], cfg["frames"], seed, cfg["sigma"])
    return topo, seg, verts


def frames_arm(args, cfg, rank, world, local_rank):
    """denoise_dynamic (denoise.hpp:258-291) through smg_denoise_dynamic: each rank
    denoises its own sequence (frame sequences are independent: weak scaling,
    no collective).  value = vertex-frames/s with device-resident frames; e2e =
    host frames in, host frames out."""
    import ctypes as C
    import numpy as np
    import torch
    import paper_1810_02719_b200 as G
    from paper_1810_02719_b200 import _abi
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    ctx = G.Context(local_rank)
    topo, seg, verts = _frames_inputs(cfg, cfg["seed0"] + rank)
    F, n, K = cfg["frames"], topo.n, seg.count
    offs, members = seg.flat()
    seq = np.arange(K, dtype=np.int32)
    d_xyz = [[torch.from_numpy(np.ascontiguousarray(v[:, a])).to(dev) for a in range(3)] for v in verts]
    h_xyz = [[torch.from_numpy(np.ascontiguousarray(v[:, a])).pin_memory() for a in range(3)] for v in verts]
    conn = dict(offs=topo.adj_offsets, cols=topo.adj_cols, moffs=offs, members=members, seq=seq)
    d_conn = {k: torch.from_numpy(np.asarray(a, np.int32)).to(dev) for k, a in conn.items()}
    h_conn = {k: torch.from_numpy(np.asarray(a, np.int32)).pin_memory() for k, a in conn.items()}
    d_out = torch.empty((F, 3 * n), dtype=torch.float64, device=dev)
    h_out = torch.empty((F, 3 * n), dtype=torch.float64).pin_memory()
    pc = _abi.smg_pipeline_config()
    ctx.lib.smg_default_config(pc)
    pc.weighting = _abi.WEIGHTING[PINNED["weighting"]]
    pc.subspace_size = cfg["c"]
    pc.iterations = cfg["t"]
    pc.power = PINNED["power"]
    pc.shift_scale = PINNED["shift_scale"]
    sizes = np.full(K, cfg["c"], np.int32)
    nb = C.c_int32()
    tms = np.zeros(3)

    def views(on):
        xyz, cn, out = (d_xyz, d_conn, d_out) if on else (h_xyz, h_conn, h_out)
        ms = (_abi.smg_mesh * F)()
        for f in range(F):
            ms[f] = _abi.smg_mesh(n, xyz[f][0].data_ptr(), xyz[f][1].data_ptr(), xyz[f][2].data_ptr(),
                                  cn["offs"].data_ptr(), cn["cols"].data_ptr(), on)
        sv = _abi.smg_segmentation(K, cn["moffs"].data_ptr(), cn["members"].data_ptr(), K, cn["seq"].data_ptr(), on)
        outp = (C.c_void_p * F)(*[out[f].data_ptr() for f in range(F)])
        return ms, sv, outp

    vw = {on: views(on) for on in (0, 1)}

    def step(on):
        ms, sv, outp = vw[on]
        ctx.check(ctx.lib.smg_denoise_dynamic(ctx.handle, F, ms, C.byref(sv), C.byref(pc), sizes.ctypes.data, 1,
                                              outp, on, C.byref(nb), tms.ctypes.data_as(_abi.c_double_p)))

    def launches():
        n_, t_ = C.c_int64(), C.c_double()
        ctx.lib.smg_profile_read(ctx.handle, b"launches", C.byref(n_), C.byref(t_))
        return n_.value

    def timed(on, steps):
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = launches()
        ev0.record()
        basis_s = frames_s = 0.0
        for _ in range(steps):
            step(on)
            basis_s += tms[0]
            frames_s += tms[1]
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        if dist is not None:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, launches() - l0, basis_s / steps, frames_s / steps

    for _ in range(args.warmup):
        step(1)
    ctx.lib.smg_profile_enable(ctx.handle, 1)
    with ClockSampler(local_rank) as clk:
        ms, nl, basis_s, frames_s = timed(1, args.steps)
    stages = {}
    for nm in ("frames", "frames_gemm", "solve", "orthonormalize", "project"):
        n_, t_ = C.c_int64(), C.c_double()
        ctx.lib.smg_profile_read(ctx.handle, nm.encode(), C.byref(n_), C.byref(t_))
        stages[nm] = {"launches": n_.value / args.steps, "ms": t_.value / args.steps}
    ctx.lib.smg_profile_enable(ctx.handle, 0)
    step(0)
    ms_e2e, _, _, _ = timed(0, args.steps)
    ms_step = ms / args.steps
    units = world * F * n
    c = cfg["c"]
    n_d = seg.block_size
    # frames-stage GEMMs: C = U^T X and X^ = U C, 2 * (2 n_d c 3F) flops per tile
    gemm_flops = K * 2 * 2.0 * n_d * c * 3 * F
    g = stages["frames_gemm"]
    achieved = gemm_flops / (g["ms"] * 1e-3) / 1e12 if g["ms"] > 0 else None
    out = {
        "metric": METRIC + " [F3 denoise_dynamic: vertex-frames/s]", "value": units / (ms_step * 1e-3),
        "unit": "vertex-frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded moving sinusoid height-field grid sequence + per-frame N(0,sigma^2) noise)",
        "config": {"workload": f"F3: {cfg['desc']}", "frames": F, "n_vertices": n, "tiles": K, "n_d": n_d, "c": c,
                   "parallelism": f"one sequence per GPU ({world} GPU(s))",
                   "l2": "frames (%.0f MB) larger than L2" % (F * n * 24 / 1e6)},
        "e2e": {"value": units / (ms_e2e / args.steps * 1e-3), "unit": "vertex-frames/s",
                "h2d_bytes_per_step": F * n * 24 + (n + 1 + len(topo.adj_cols) + K * n_d + 2 * (K + 1)) * 4,
                "d2h_bytes_per_step": F * n * 24},
        "roofline": {"kernel": "frames-stage DMMA GEMMs (U^T X, U C over 3F frame columns)", "bound": "tensor",
                     "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS if achieved else None, "traffic": None,
                     "flops_per_step": gemm_flops, "gemm_ms_per_step": g["ms"], "launches_per_step": g["launches"]},
        "split_ms": {"shared_basis": basis_s * 1e3, "frames": frames_s * 1e3},
        "frames_stage_value": units / frames_s if frames_s > 0 else None,
        "stages_ms_per_step": {k: round(v["ms"], 3) for k, v in stages.items()},
        "clocks": clk.summary(), "gpu_launches": nl,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = frames_cpu_baseline(args, cfg)
    if dist is not None:
        dist.destroy_process_group()
    ctx.close()
    return out if rank == 0 else None


def frames_cpu_baseline(args, cfg):
    """The oracle's denoise_dynamic on a bounded sample: the chain over the first T
    tiles, then all F frames projected onto those T bases, extrapolated to all
    tiles (one core, BLAS 1 thread -- the reference's frames loop is parallel_for
    over frames, so the frames share is divided by the host cores)."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import specmesh_oracle as O
    cores = os.cpu_count() or 1
    topo, seg, verts = _frames_inputs(cfg, cfg["seed0"])
    T = min(seg.count, max(2, args.cpu_tiles))
    subs = O.build_submeshes(topo.adj_offsets, topo.adj_cols, seg.members[:T])
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=cfg["c"], iterations=cfg["t"],
                            shift_scale=PINNED["shift_scale"])
    t0 = time.perf_counter()
    bb = O.compute_block_bases_fixed_sizes(verts[0], subs, np.arange(T), ocfg, [cfg["c"]] * T)
    t1 = time.perf_counter()
    for v in verts:
        O.project_blocks(bb, v)
    t2 = time.perf_counter()
    K, F, n = seg.count, cfg["frames"], topo.n
    t_step = (t1 - t0) * K / T + (t2 - t1) * K / T / cores
    return {"value": F * n / t_step, "unit": "vertex-frames/s", "cores": cores, "kind": "port",
            "sample": f"chain over the first {T} of {K} tiles ({t1 - t0:.2f}s, 1 core) + {F} frames projected on "
                      f"those tiles ({t2 - t1:.2f}s, 1 core; frames loop credited with {cores} cores), "
                      f"extrapolated to {K} tiles"}


def frames_reference_arm(args, cfg):
    vals = []
    for _ in range(max(1, args.steps)):
        cb = frames_cpu_baseline(args, cfg)
        vals.append(cb["value"])
    cb["value"] = statistics.median(vals)
    units = cfg["frames"] * cfg["W"] * cfg["H"]
    return {"metric": METRIC + " [F3 denoise_dynamic: vertex-frames/s]", "value": cb["value"],
            "unit": "vertex-frames/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": units / cb["value"] * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"F3: {cfg['desc']}"}, "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "vertex-frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


# ----------------------------------------------------------------------- F4 arm

def _fine_inputs(cfg, seed):
    from paper_1810_02719_b200 import synth
    return synth.grid_mesh(cfg["W"], cfg["H"], seed, cfg["sigma"])


def fine_arm(args, cfg, rank, world, local_rank):
    """fine_denoise (denoise.hpp:172-178) through smg_fine_denoise; one mesh per
    rank (independent meshes: weak scaling, no collective)."""
    import ctypes as C
    import numpy as np
    import torch
    import paper_1810_02719_b200 as G
    from paper_1810_02719_b200 import _abi
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    ctx = G.Context(local_rank)
    m = _fine_inputs(cfg, cfg["seed0"] + rank)
    n, nf = m.n, m.faces.shape[0]
    d_xyz = [torch.from_numpy(np.ascontiguousarray(m.vertices[:, a])).to(dev) for a in range(3)]
    h_xyz = [torch.from_numpy(np.ascontiguousarray(m.vertices[:, a])).pin_memory() for a in range(3)]
    d_f = torch.from_numpy(np.ascontiguousarray(m.faces, dtype=np.int32)).to(dev)
    h_f = torch.from_numpy(np.ascontiguousarray(m.faces, dtype=np.int32)).pin_memory()
    d_out = torch.empty(3 * n, dtype=torch.float64, device=dev)
    h_out = torch.empty(3 * n, dtype=torch.float64).pin_memory()
    bp = _abi.smg_bilateral_params()
    ctx.lib.smg_default_bilateral_params(C.byref(bp))

    def step(on):
        xyz, f, out = (d_xyz, d_f, d_out) if on else (h_xyz, h_f, h_out)
        ctx.check(ctx.lib.smg_fine_denoise(ctx.handle, n, xyz[0].data_ptr(), xyz[1].data_ptr(), xyz[2].data_ptr(), nf,
                                           f.data_ptr(), C.byref(bp), out.data_ptr(), None, on))

    def launches():
        n_, t_ = C.c_int64(), C.c_double()
        ctx.lib.smg_profile_read(ctx.handle, b"launches", C.byref(n_), C.byref(t_))
        return n_.value

    def timed(on, steps):
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = launches()
        ev0.record()
        for _ in range(steps):
            step(on)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        if dist is not None:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, launches() - l0

    for _ in range(args.warmup):
        step(1)
    ctx.lib.smg_profile_enable(ctx.handle, 1)
    with ClockSampler(local_rank) as clk:
        ms, nl = timed(1, args.steps)
    stages = {}
    for nm in ("fine_geometry", "fine_rings", "fine_sigma", "fine_normals", "fine_vertices"):
        n_, t_ = C.c_int64(), C.c_double()
        ctx.lib.smg_profile_read(ctx.handle, nm.encode(), C.byref(n_), C.byref(t_))
        stages[nm] = t_.value / args.steps
    ctx.lib.smg_profile_enable(ctx.handle, 0)
    step(0)
    ms_e2e, _ = timed(0, args.steps)
    ms_step = ms / args.steps
    units = world * n
    # dominant kernel: the bilateral sweep; algorithmic bytes per face and sweep =
    # its {centroid, area} + normal read (2 x 32 B) + normal write (32 B) + ring
    # offsets (4 B) + ring ids (4 B per member, 13 on this grid: 52 B) = 152 B
    ring_ids = 13
    bytes_face = 32 + 32 + 32 + 4 + 4 * ring_ids
    sweeps = bp.normal_iterations
    t_sweep = stages["fine_normals"] / sweeps if stages["fine_normals"] > 0 else None
    achieved = bytes_face * nf / (t_sweep * 1e-3) / 1e9 if t_sweep else None
    peak = 6550.7
    try:
        with open(PEAKS) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass
    out = {
        "metric": METRIC + " [F4 fine_denoise: vertices/s]", "value": units / (ms_step * 1e-3), "unit": "vertices/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded sinusoid height-field grid + N(0, 0.01^2) noise)",
        "config": {"workload": f"F4: {cfg['desc']}", "vertices": n, "faces": nf,
                   "params": {"sigma_spatial": "auto", "sigma_range": bp.sigma_range,
                              "normal_iterations": bp.normal_iterations,
                              "vertex_iterations": bp.vertex_iterations, "ring_depth": bp.ring_depth},
                   "parallelism": f"one mesh per GPU ({world} GPU(s))",
                   "l2": "face data (%.0f MB) larger than L2" % (nf * 64 / 1e6)},
        "e2e": {"value": units / (ms_e2e / args.steps * 1e-3), "unit": "vertices/s",
                "h2d_bytes_per_step": 3 * n * 8 + nf * 12, "d2h_bytes_per_step": 3 * n * 8},
        "roofline": {"kernel": "bilateral_kernel (one Jacobi sweep of the normal filter)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None, "traffic": None,
                     "bytes_per_face": bytes_face, "sweep_ms": t_sweep,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
        "stages_ms_per_step": {k: round(v, 3) for k, v in stages.items()},
        "clocks": clk.summary(), "gpu_launches": nl,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = fine_cpu_baseline(cfg)
    if dist is not None:
        dist.destroy_process_group()
    ctx.close()
    return out if rank == 0 else None


def fine_cpu_baseline(cfg, rows=128):
    """The oracle's fine_denoise on a bounded sample: the first `rows` grid rows
    (a W x rows strip, same connectivity pattern), one core, scaled per vertex."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import specmesh_oracle as O
    from paper_1810_02719_b200 import synth
    m = synth.grid_mesh(cfg["W"], rows, cfg["seed0"], cfg["sigma"])
    t0 = time.perf_counter()
    O.fine_denoise(m.vertices, m.faces, O.BilateralParams())
    dt = time.perf_counter() - t0
    return {"value": m.n / dt, "unit": "vertices/s", "cores": 1, "kind": "port",
            "sample": f"oracle fine_denoise of a {cfg['W']} x {rows} strip of the grid ({m.n} vertices, "
                      f"{dt:.2f}s, numpy vectorised over faces, 1 core)"}


def fine_reference_arm(args, cfg):
    vals = [fine_cpu_baseline(cfg)["value"] for _ in range(max(1, args.steps))]
    cb = fine_cpu_baseline(cfg)
    cb["value"] = statistics.median(vals)
    units = cfg["W"] * cfg["H"]
    return {"metric": METRIC + " [F4 fine_denoise: vertices/s]", "value": cb["value"], "unit": "vertices/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": units / cb["value"] * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": {"workload": f"F4: {cfg['desc']}"},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "vertices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        arm = frames_reference_arm if "frames" in cfg else (fine_reference_arm if "fine" in cfg else reference_arm)
        print(json.dumps(arm(args, cfg)), flush=True)
        return
    if "fine" in cfg:
        if args.impl == "ours":
            out = fine_arm(args, cfg, rank, world, local_rank)
            if out is not None:
                print(json.dumps(out), flush=True)
        return
    if "frames" in cfg:
        if args.impl == "ours":
            out = frames_arm(args, cfg, rank, world, local_rank)
            if out is not None:
                print(json.dumps(out), flush=True)
        return
    out = gpu_arm(args, cfg, rank, world, local_rank)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
