#!/usr/bin/env python3
"""bench.py -- vertices/s through OI track + project + reconstruct (BASELINE.json).

Default workload: config 5 (64 independent 512x512 grid meshes, 128 tiles of
32x64 = 2048 vertices each, c = 200, one warm-started OI step per tile, fp64),
the batched configuration the metric's multi-GPU scaling is quoted on.  One
"step" = every mesh of the job carried through the full chain: Laplacian
assembly, factorisation, first-submesh basis, OI tracking, projection, stitched
reconstruction (+ the NCCL gather of per-mesh results to all ranks when N > 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1|C2|C3|C4|C5|F3|F4]
  python bench.py --impl reference ...     # CPU oracle (port) arm

`--gpus N` (N > 1) re-launches itself under torch.distributed.run with N
ranks.  Chains shard across ranks with no data-path collective.  Default: the
literal config 5 -- its 64 meshes split over the N GPUs (strong scaling);
at N > 1 the same run also measures weak scaling (every GPU a 64-mesh shard,
mesh ids rank*64 .., each its own seed) as `weak_scaling`; `--weak` makes that
the headline.  The per-mesh reconstructions are all-gathered (NCCL over
NVLink) at the end of every step.  Timing: W untimed warm-up steps, then K steps
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
    # single chains (replicas only across GPUs)
    "C1": dict(W=32, H=32, tw=32, th=32, c=40, t=10, meshes=1, single=True, seed0=101,
               desc="one 32x32 grid submesh (n_d=1024): bottom_subspace(40) + orthogonal_iteration(op, init, 10) + "
                    "gft/igft, composed from the C-ABI primitives (SURVEY.md §3.3)"),
    "C3": dict(W=0, H=0, tw=0, th=0, c=60, t=1, meshes=1, synth="C3", seed0=303,
               desc="icosphere level 7 (163 842 vertices), 160 polar-band blocks (n_d=1026), c=60, t=1, "
                    "low-pass reconstruction"),
    "C4": dict(W=1024, H=1024, tw=64, th=64, c=20, t=0, meshes=1, synth="C4", doi=True, seed0=404,
               desc="1024^2 grid, 256 tiles of 64x64 (n_d=4096), DOI c in [20, 400], band 1e-5/1e-4"),
}
PINNED = dict(weighting="binary", power=2, shift_scale=1e-3, dense_limit=4096)
DOI = dict(c_min=20, c_max=400, eps_low=1e-5, eps_high=1e-4)  # C4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--meshes", type=int, default=0, help="override the per-GPU mesh count (debug)")
    ap.add_argument("--strong", action="store_true",
                    help="(default) split the config's 64 meshes over the GPUs: the literal C5 (strong scaling)")
    ap.add_argument("--weak", action="store_true",
                    help="every GPU carries the config's full mesh count (weak scaling); at N > 1 the default "
                         "run also reports this as `weak_scaling`")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tiles", type=int, default=8, help="tiles per chain in the CPU sample")
    return ap.parse_args()


# ----------------------------------------------------------------------- inputs

def build_inputs(cfg, mesh_ids):
    """(topology mesh, segmentation, per-chain vertices, member offsets, members).
    Grid configs share one topology (each mesh its own seeded surface);
    C3 / C4 come from synth.config (the parity tests' inputs)."""
    import numpy as np
    from paper_1810_02719_b200 import synth
    if "synth" in cfg:
        w = synth.config(cfg["synth"])
        base, seg, verts = w.mesh, w.seg, [w.mesh.vertices for _ in mesh_ids]
    else:
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
        self.doi = bool(cfg.get("doi"))
        c = cfg["c"] if not self.doi else min(DOI["c_max"], self.nd)  # coefficient capacity
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
        self.sizes_out = [np.zeros(self.K, np.int32) for _ in range(self.B)]
        self.iters_out = [np.zeros(self.K, np.int32) for _ in range(self.B)]
        self.coef_off = [np.zeros(self.K + 1, np.int64) for _ in range(self.B)]
        self.sizes = np.full(self.K, c, np.int32)
        self.pcfg = _abi.smg_pipeline_config()
        ctx.lib.smg_default_config(self.pcfg)
        self.pcfg.weighting = _abi.WEIGHTING[PINNED["weighting"]]
        self.pcfg.subspace_size = c
        self.pcfg.iterations = cfg["t"]
        self.pcfg.power = PINNED["power"]
        self.pcfg.shift_scale = PINNED["shift_scale"]
        if self.doi:
            self.pcfg.subspace_size = cfg["c"]
            self.pcfg.basis_mode = _abi.BASIS_MODE["doi"]
            self.pcfg.c_min, self.pcfg.c_max = DOI["c_min"], DOI["c_max"]
            self.pcfg.eps_low, self.pcfg.eps_high = DOI["eps_low"], DOI["eps_high"]
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
            o.subspace_size = self.sizes_out[b].ctypes.data
            o.residual_rms = st[1].ctypes.data
            o.doi_residual = st[2].ctypes.data
            o.converged = None
            o.oi_iterations = self.iters_out[b].ctypes.data
            o.reconstruction = recon[b].data_ptr()
            o.coefficients = coef[b].data_ptr()
            o.coefficients_capacity = self.ncoef
            o.coefficient_offsets = self.coef_off[b].ctypes.data
            o.on_device = on_device
        return meshes, segs, outs

    def run(self, on_device):
        meshes, segs, outs = self.views[on_device]
        if self.doi:  # compute_block_bases, DOI branch (one chain)
            st = self.ctx.lib.smg_compute_block_bases(self.ctx.handle, meshes, segs, self.pcfg, outs)
        else:
            st = self.ctx.lib.smg_run_chains(self.ctx.handle, self.B, meshes, segs, self.pcfg,
                                             self.sizes.ctypes.data, outs)
        self.ctx.check(st)


def _solve_flops(cfg, job, trajectory, W_used):
    """Algorithmic and executed flops of one step's solve
    launches: z*4*n_d*b*c per tile and OI step with b the natural-order
    half-bandwidth, + the first basis's shift-invert bootstrap (4 iterations on
    m columns, the first with z = 1).  The executed count is the block solve's
    own, 3*n*W*cols per triangular sweep (2z sweeps per step) at the block
    width the library chose.  `trajectory`: per chain, the c of every OI step."""
    n, z = job.nd, PINNED["power"]
    b_half = (cfg["tw"] + 1) if cfg["tw"] else 33  # C3: 33 nominal
    c0 = cfg["c"]
    m_fb = min(n, max(c0, min(480, -(-(c0 + max(16, c0 // 6)) // 8) * 8)))
    cols = sum(sum(tr) for tr in trajectory)
    alg = z * 4.0 * n * b_half * cols + job.B * (1 + 3 * z) * 4.0 * n * b_half * m_fb
    hw = 3.0 * n * W_used * (2 * z * cols + job.B * (2 + 3 * 2 * z) * m_fb)
    return alg, hw, b_half


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
    ctx = G.Context(local_rank)
    comm = None
    if dist is not None and cfg["meshes"] > 1:
        # the library's NCCL communicator (smg_comm_create): the per-mesh gather
        # runs in the C++ host, the process group only broadcasts the unique id
        comm = shard.LibComm(ctx, world, rank, broadcast=shard.torch_broadcast)
    args._comm = comm
    out = measure_job(args, cfg, rank, world, local_rank, ctx, dist, weak=args.weak)
    if out is not None and world > 1 and cfg["meshes"] > 1 and not args.weak:
        # the second scaling mode on the same ranks: every GPU carries a full
        # 64-mesh shard (weak scaling); the headline stays the literal config
        w = measure_job(args, cfg, rank, world, local_rank, ctx, dist, weak=True, brief=True)
        if w is not None:
            out["weak_scaling"] = w
    elif world > 1 and cfg["meshes"] > 1 and not args.weak:
        measure_job(args, cfg, rank, world, local_rank, ctx, dist, weak=True, brief=True)
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()
    ctx.close()
    return out if rank == 0 else None


def measure_job(args, cfg, rank, world, local_rank, ctx, dist, weak=False, brief=False):
    import numpy as np
    import torch
    from paper_1810_02719_b200 import shard
    per_gpu = args.meshes or cfg["meshes"]
    total_meshes = per_gpu * world if weak else per_gpu
    if cfg["meshes"] == 1:  # single-chain configs: replicas only
        ids = [rank]
        total_units = world
    else:
        ids = shard.shard_meshes(total_meshes, world, rank)
        total_units = total_meshes
    job = GpuJob(cfg, ids, local_rank, ctx)
    verts_per_unit = job.n
    gather = dist is not None and cfg["meshes"] > 1
    comm = getattr(args, "_comm", None)
    gathered = torch.empty((total_meshes, 3 * job.n), dtype=torch.float64, device=job.dev) if gather else None

    def step(on_device):
        job.run(on_device)
        if gather and on_device:
            # per-mesh reconstructions to every rank: smg_gather_meshes (NCCL
            # all-gather over NVLink, ragged shards padded in the library)
            if comm is not None:
                comm.gather(job.d_recon, gathered, total_meshes, 3 * job.n)
                torch.cuda.synchronize()
            else:
                shard.gather_meshes(job.d_recon, total_meshes)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def launches():
        import ctypes as C
        n, t = C.c_int64(), C.c_double()
        ctx.lib.smg_profile_read(ctx.handle, b"launches", C.byref(n), C.byref(t))
        return n.value

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

    # untimed: the run's choices and (DOI) the c of every step
    if job.doi:
        ctx.doi_trace(True)
        job.run(True)
        _, c_steps, _ = ctx.read_doi_trace()
        ctx.doi_trace(False)
        trajectory = [list(map(int, c_steps))]
    else:
        job.run(True)
        trajectory = [[cfg["c"]] * ((job.K - 1) * cfg["t"])] * job.B
    info = ctx.last_run_info()
    for _ in range(max(0, args.warmup - 1)):
        step(True)
    with ClockSampler(local_rank) as clk:
        ms, nl = timed(True, args.steps, profile=True)
    clocks = clk.summary()
    stages = {}
    import ctypes as C
    for nm in ("assemble", "factor", "first_basis", "fb_iterate", "fb_filter", "fb_rayleigh_ritz", "solve",
               "orthonormalize", "gram", "chol", "trmm", "project"):
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
    scaling = "weak" if (weak or cfg["meshes"] == 1) else "strong"
    if brief:
        return {"value": value, "unit": "vertices/s", "ms_per_step": ms_step, "scaling": scaling,
                "meshes": total_units, "meshes_per_gpu": len(ids),
                "e2e": {"value": e2e_value, "unit": "vertices/s"}, "clocks": clocks}

    # roofline of the dominant kernel (solve: the block-tridiagonal R^z sweeps).
    # Launch durations are CUDA-event spans on the launching stream inside the
    # timed region; with two chain groups a launch's span includes time the
    # other group's kernels occupy SMs.
    W_used = info["block_width"]
    alg, hw, b_half = _solve_flops(cfg, job, trajectory, W_used)
    solve = stages["solve"]
    kernel = "solve_kernel (block-tridiagonal R^z sweeps, DMMA f64)"
    if job.doi and not solve["ms"]:
        # the DOI loop is one captured graph per block (solve -> CholeskyQR2 ->
        # residual -> decide): its kernels are not profiled one by one, so the
        # roofline is the whole step's OI work over the step time
        kernel = "DOI step graph (solve + CholeskyQR2 + residual per step), whole step"
        n_, z_ = job.nd, PINNED["power"]
        alg = sum(z_ * 4.0 * n_ * b_half * cc + 4.0 * n_ * cc * cc for tr in trajectory for cc in tr)
        solve = {"ms": ms_step, "launches": args.steps}
    spl = solve["launches"] / args.steps if solve["launches"] else 0
    achieved = alg / (solve["ms"] * 1e-3) / 1e12 if solve["ms"] > 0 else None
    traffic = None
    try:  # dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "solve_traffic_r02.json")) as f:
            traffic = json.load(f)["dram_bytes_per_launch"] if args.config == "C5" else None
    except (OSError, KeyError, ValueError):
        pass
    roofline = {"kernel": kernel, "bound": "tensor",
                "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None, "traffic": traffic,
                "traffic_source": "profiles/solve_traffic_r02.json (bytes per launch of 32 chains)",
                "peak_source": "measured FP64 DMMA peak, profiles/fp64_peak_r01.txt (MEASURED_PEAKS.json has no FP64 entry)",
                "flops_per_launch": alg / max(spl, 1e-9), "avg_launch_ms": solve["ms"] / max(spl, 1e-9),
                "b_algorithmic": b_half, "block_width_used": W_used, "ordering": info["ordering"],
                "hw_flops_per_launch": hw / max(spl, 1e-9),
                "hw_frac": (hw / (solve["ms"] * 1e-3) / 1e12 / FP64_PEAK_TFLOPS) if solve["ms"] > 0 else None,
                "launches_per_step": spl,
                "step_share": solve["ms"] / ms_step if ms_step else None}
    # whole-step algorithmic FP64 work (SURVEY.md §8(d) formulas, per GPU)
    # z*4*n*b*c + 4*n*c^2 per OI step, n*b^2 + 12*n*c + 3*n per tile, (4/3)n^3 + 2n^2c first tile
    n, z, c = job.nd, PINNED["power"], cfg["c"]
    oi = sum(z * 4.0 * n * b_half * cc + 4.0 * n * cc * cc for tr in trajectory for cc in tr)
    c_tiles = sum(int(v) for s in job.sizes_out for v in s) if job.doi else job.B * job.K * c
    tiles = job.B * job.K * (n * b_half ** 2 + 3.0 * n) + 12.0 * n * c_tiles
    first = job.B * ((4.0 / 3.0) * n ** 3 + 2.0 * n * n * c)
    step_flops = oi + tiles + first
    # steady state: the chain without its first-submesh basis
    fb_ms = stages["first_basis"]["ms"]
    steady = units * (job.K - 1) / job.K / ((ms_step - fb_ms) / 1e3) if ms_step > fb_ms > 0 else None
    out = {
        "metric": METRIC, "value": value, "unit": "vertices/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded sinusoid height-field grids / icosphere + noise; no dataset exists)",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "meshes": total_units, "meshes_per_gpu": len(ids),
                   "tiles_per_mesh": job.K, "n_d": n, "c": c if not job.doi else "DOI [20, 400]",
                   "oi_iterations": cfg["t"], "z": z, "shift_scale": PINNED["shift_scale"],
                   "weighting": PINNED["weighting"], "tile_order": "row-major" if cfg["tw"] else "partition order",
                   "parallelism": (f"chains sharded over {world} GPU(s), "
                                   + (f"{len(ids)} meshes per GPU (weak)" if weak
                                      else f"{total_meshes} meshes split (strong)")) if cfg["meshes"] > 1
                   else "replicas",
                   "l2": "inputs larger than L2 (%.0f MB per GPU)" % (job.h2d_bytes / 1e6)},
        "e2e": {"value": e2e_value, "unit": "vertices/s", "h2d_bytes_per_step": job.h2d_bytes,
                "d2h_bytes_per_step": job.d2h_bytes},
        "roofline": roofline,
        "steady_state": {"value": steady, "unit": "vertices/s",
                         "note": "chain without the first-submesh basis (its device time subtracted)"},
        "fp64_step_efficiency": {"algorithmic_tflop_per_step": step_flops / 1e12,
                                 "achieved_tflops": step_flops / (ms_step * 1e-3) / 1e12,
                                 "frac_of_peak": step_flops / (ms_step * 1e-3) / 1e12 / FP64_PEAK_TFLOPS},
        "stages_ms_per_step": {k: round(v["ms"], 3) for k, v in stages.items()},
        "run_info": info,
        "clocks": clocks,
        "gpu_launches": nl,
    }
    if job.doi:
        out["config"]["doi_steps"] = len(trajectory[0])
        out["config"]["c_final"] = {"min": int(job.sizes_out[0].min()), "max": int(job.sizes_out[0].max())}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, cfg, total_units)
    return out if rank == 0 else None


def single_arm(args, cfg, rank, world, local_rank):
    """C1: the reference has no single-call entry; the path is
    the composition build_laplacian -> ShiftedInverseOperator ->
    bottom_subspace(c) -> orthogonal_iteration(op, init, 10) -> gft / igft,
    here through the C-ABI primitives (host pointers: every call copies its
    inputs in and its results out, so `value` already includes the copies and
    equals `e2e`).  Replicas only across GPUs."""
    import ctypes as C
    import numpy as np
    import torch
    import paper_1810_02719_b200 as G
    from paper_1810_02719_b200 import synth
    torch.cuda.set_device(local_rank)
    ctx = G.Context(local_rank)
    w = synth.config(args.config)
    mem = np.sort(w.seg.members[0])
    x = w.mesh.vertices[mem]
    n = int(mem.size)

    def step():
        rp, cols, vals, tr = G.build_laplacian(w.mesh, mem, weighting="binary", ctx=ctx)
        op = G.ShiftedInverseOperator(rp, cols, vals, G.default_shift(tr, n, PINNED["shift_scale"]), PINNED["power"],
                                      ctx=ctx)
        u = G.orthogonal_iteration(op, G.bottom_subspace(op, cfg["c"]), cfg["t"])
        return G.igft(u, G.gft(u, x, ctx=ctx), ctx=ctx)

    def launches():
        nn, t = C.c_int64(), C.c_double()
        ctx.lib.smg_profile_read(ctx.handle, b"launches", C.byref(nn), C.byref(t))
        return nn.value

    for _ in range(max(1, args.warmup)):
        step()
    ctx.lib.smg_profile_enable(ctx.handle, 1)
    l0 = launches()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
    ms_step = ev0.elapsed_time(ev1) / args.steps
    nl = launches() - l0
    stages = {}
    for nm in ("assemble", "factor", "first_basis", "solve", "orthonormalize", "gram", "chol", "trmm", "project"):
        nn, t = C.c_int64(), C.c_double()
        ctx.lib.smg_profile_read(ctx.handle, nm.encode(), C.byref(nn), C.byref(t))
        stages[nm] = round(t.value / args.steps, 3)
    ctx.lib.smg_profile_enable(ctx.handle, 0)
    ctx.close()
    z, c, t = PINNED["power"], cfg["c"], cfg["t"]
    b_half = cfg["tw"] + 1
    oi_flops = t * (z * 4.0 * n * b_half * c + 4.0 * n * c * c)
    value = world * n / (ms_step / 1e3)
    h2d = x.nbytes + mem.nbytes + w.mesh.adj_offsets.nbytes + w.mesh.adj_cols.nbytes + w.mesh.vertices.nbytes
    out = {"metric": METRIC, "value": value, "unit": "vertices/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded sinusoid height-field grid)",
           "config": {"workload": f"{args.config}: {cfg['desc']}", "n_d": n, "c": c, "oi_iterations": t, "z": z,
                      "shift_scale": PINNED["shift_scale"], "parallelism": "replicas",
                      "l2": "tiny single submesh (latency-bound)"},
           "e2e": {"value": value, "unit": "vertices/s", "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(n * 3 * 8 * 2 + c * 3 * 8)},
           "roofline": {"kernel": "the 10 OI steps (solve + CholeskyQR2)", "bound": "tensor",
                        "achieved": oi_flops / ((stages["solve"] + stages["orthonormalize"]) * 1e-3) / 1e12
                        if stages["solve"] > 0 else None,
                        "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                        "frac": oi_flops / ((stages["solve"] + stages["orthonormalize"]) * 1e-3) / 1e12
                        / FP64_PEAK_TFLOPS if stages["solve"] > 0 else None, "traffic": None,
                        "note": "one 1024 x 40 block: latency-bound (a few CTAs); frac of the whole GPU's peak"},
           "stages_ms_per_step": stages, "clocks": clk.summary(), "gpu_launches": nl}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, cfg, 1)
    return out if rank == 0 else None


# ----------------------------------------------------------------------- CPU arm

_CPU_STATE = {}


def _cpu_worker_init():
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _cpu_prepare(task):
    """Untimed: build one chain's inputs in the worker (mesh, submeshes)."""
    cfgname, mesh_id = task
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import specmesh_oracle as O
    from paper_1810_02719_b200 import synth
    cfg = CONFIGS[cfgname]
    if "synth" in cfg or cfg.get("single"):
        w = synth.config(cfgname)
        base, seg = w.mesh, w.seg
    else:
        base = synth.grid_mesh(cfg["W"], cfg["H"], cfg["seed0"] + mesh_id, cfg["sigma"])
        seg = synth.grid_tiles(cfg["W"], cfg["H"], cfg["tw"], cfg["th"])
    subs = O.build_submeshes(base.adj_offsets, base.adj_cols, seg.members)
    _CPU_STATE[task] = (base, seg, subs)
    return os.getpid()


def _cpu_chain(task):
    """One whole chain of the oracle port, timed like the reference's
    StageTimings (core.hpp:57-68): track + project + reconstruct.  Returns
    (chain seconds, first-basis seconds, vertices)."""
    import numpy as np
    import specmesh_oracle as O
    O.ShiftedInverseOperator.rcm_above = 0  # bandwidth-minimising order, as the GPU's geometric ordering
    cfgname, mesh_id = task
    if task not in _CPU_STATE:
        _cpu_prepare(task)
    base, seg, subs = _CPU_STATE[task]
    cfg = CONFIGS[cfgname]
    if cfg.get("single"):
        # C1: build_laplacian -> operator -> dense eig + bottom_subspace
        # -> orthogonal_iteration(op, init, t) -> gft / igft
        t0 = time.perf_counter()
        lap = O.build_laplacian(subs[0], base.vertices, O.BINARY)
        op = O.ShiftedInverseOperator(lap, O.default_shift(lap, PINNED["shift_scale"]), PINNED["power"])
        init = O.bottom_subspace(O.dense_eigendecomposition(lap), cfg["c"])
        t1 = time.perf_counter()
        u = O.orthogonal_iteration(op, init, cfg["t"])
        O.igft(u, O.gft(u, subs[0].local_coords(base.vertices)))
        t2 = time.perf_counter()
        return t2 - t0, t1 - t0, base.n
    t0 = time.perf_counter()
    if cfg.get("doi"):
        ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=cfg["c"], shift_scale=PINNED["shift_scale"], **DOI)
        bb = O.compute_block_bases_doi(base.vertices, subs, seg.sequence, ocfg)
        fb = 0.0
    else:
        ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=cfg["c"], iterations=cfg["t"],
                                shift_scale=PINNED["shift_scale"])
        bb = O.compute_block_bases_fixed_sizes(base.vertices, subs, seg.sequence, ocfg, [cfg["c"]] * seg.count)
        fb = bb.timings.get("first_basis", 0.0)
    O.reconstruct_weighted(subs, O.project_blocks(bb, base.vertices), base.n)
    t1 = time.perf_counter()
    return t1 - t0, fb, base.n


class CpuArm:
    """The oracle port on the host cores: one whole chain per core (BLAS 1
    thread), the reference's only concurrency (detail::parallel_for,
    core.hpp:84-100).  A step = P whole chains; its time = the slowest chain."""

    def __init__(self, cfgname, P, first_mesh=0):
        import multiprocessing as mp
        for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[k] = "1"
        self.cfgname, self.P = cfgname, P
        self.tasks = [(cfgname, first_mesh + i) for i in range(P)]
        # one single-process pool per chain (a chain never shares a core or
        # moves between workers); fresh interpreters that read the 1-thread
        # BLAS settings at import; inputs prepared untimed
        ctxm = mp.get_context("spawn")
        self.pools = [ctxm.Pool(1, initializer=_cpu_worker_init) for _ in range(P)]
        for r in [pl.apply_async(_cpu_prepare, (t,)) for pl, t in zip(self.pools, self.tasks)]:
            r.get()

    def step(self):
        res = [r.get() for r in [pl.apply_async(_cpu_chain, (t,)) for pl, t in zip(self.pools, self.tasks)]]
        return max(r[0] for r in res), sum(r[2] for r in res), statistics.mean(r[1] for r in res)

    def close(self):
        for pl in self.pools:
            pl.close()
        for pl in self.pools:
            pl.join()


def cpu_baseline(args, cfg, total_units):
    """Rank 0, N=1: one step of the CPU arm (bounded: P whole chains on P cores)."""
    cores = os.cpu_count() or 1
    P = min(cores, max(1, total_units))
    arm = CpuArm(args.config, P)
    try:
        t, verts, tfb = arm.step()
    finally:
        arm.close()
    out = {"value": verts / t, "unit": "vertices/s", "cores": P, "kind": "port",
            "steady_state_value": verts / (t - tfb) if t > tfb else None,
            "sample": f"{P} whole chains ({cfg['desc']}) in parallel, 1 per core, BLAS 1 thread; numpy/LAPACK "
                      f"restatement oracle/specmesh_oracle.py (pinned to the reference's own code run over an Eigen stand-in, "
                      f"tests/golden/ref_*; that build is slower than LAPACK, so the port is the baseline); banded Cholesky at the bandwidth-minimising order (RCM, "
                      f"b=33 like the GPU); timed track+project+reconstruct per chain, no extrapolation; "
                      f"step {t:.1f}s, first basis {tfb:.1f}s per chain"}
    ref = reference_code_sample(args)
    if ref:
        out["reference_code"] = ref
    return out


def reference_code_sample(args, tiles=32):
    """The reference's OWN chain code (its headers over oracle/eigen_shim, built where
    /root/reference exists and shipped as oracle/_ref/libspecmesh_ref.so) on a bounded sample:
    the first `tiles` tiles of one C5 chain on one core, tracking only (the first-submesh
    eigendecomposition excluded).  A cross-check of the port's baseline, not the baseline: the
    stand-in's unblocked QR / LDL^T are slower than LAPACK (and than real Eigen)."""
    if args.config != "C5":
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import numpy as np
        import ref_binding as R
        if not R.available():
            return None
        from paper_1810_02719_b200 import synth
        w = synth.config("C5", mesh_index=0)
        rm = R.Mesh(w.mesh.vertices, w.mesh.faces)
        # dense_limit below n_d: the first tile starts from the reference's cold random basis with one
        # OI step (pipeline.hpp:118-119) instead of the n_d^3 dense eigendecomposition, so the sample
        # times tracking steps only (their cost does not depend on the basis values)
        cfg = R.default_config(weighting=R.BINARY, subspace_size=w.c, iterations=w.iterations, shift_scale=1e-3,
                               dense_limit=16, initial_iterations=1)
        rs = R.Segmentation.from_members(rm, w.seg.members[:tiles], np.arange(tiles, dtype=np.int32))
        t0 = time.perf_counter()
        R.chain_fixed(rm, rs, cfg, [w.c] * tiles)
        per_tile = (time.perf_counter() - t0) / tiles
        n_d = int(w.seg.members[0].size)
        return {"value": n_d / per_tile, "unit": "vertices/s", "cores": 1, "seconds_per_tile": per_tile,
                "sample": f"compute_block_bases_fixed_sizes (pipeline.hpp:144-194) of the reference itself over "
                          f"oracle/eigen_shim on {tiles} tiles of C5 mesh 0 (cold-start first tile, no dense "
                          f"eigendecomposition), one core, tracking steps only"}
    except Exception as exc:  # the cross-check never fails the bench
        return {"unavailable": f"{type(exc).__name__}: {exc}"}


def reference_arm(args, cfg):
    """--impl reference: the oracle port on all host cores.  Each step = P
    whole chains (P = host cores, capped at the job's mesh count); the rate is
    vertices processed / slowest chain.  One warm-up step at most (the CPU has
    no caches to warm beyond the first call's imports)."""
    total_units = (args.meshes or cfg["meshes"]) * (max(1, args.gpus) if args.weak else 1)
    cores = os.cpu_count() or 1
    P = min(cores, max(1, total_units))
    arm = CpuArm(args.config, P)
    t_start = time.perf_counter()
    try:
        for _ in range(min(args.warmup, 1)):
            arm.step()
        times, verts, tfbs = [], 0, []
        for _ in range(max(1, args.steps)):
            t, v, tfb = arm.step()
            times.append(t)
            tfbs.append(tfb)
            verts = v
            if time.perf_counter() - t_start > 150:  # bounded: the run stays within a few minutes (C4: one chain)
                break
    finally:
        arm.close()
    total_t = sum(times)
    value = verts * len(times) / total_t
    steady = verts * len(times) / (total_t - sum(tfbs))
    ms_step = total_t / len(times) * 1e3
    cb = {"value": value, "unit": "vertices/s", "cores": P, "kind": "port", "steady_state_value": steady,
          "sample": f"per step {P} whole chains of {args.config} in parallel (1 per core, BLAS 1 thread), "
                    f"numpy/LAPACK restatement oracle/specmesh_oracle.py; no extrapolation"}
    return {"metric": METRIC, "value": value, "unit": "vertices/s", "n_gpus": args.gpus, "steps": len(times),
            "warmup": min(args.warmup, 1), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if (args.weak or cfg["meshes"] == 1) else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded sinusoid height-field grids + N(0,sigma^2) noise)",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "meshes_per_step": P,
                       "job_meshes": total_units},
            "impl": "reference", "arm": "oracle port (numpy/LAPACK restatement of the reference, pinned to the reference's own code over an Eigen stand-in; Eigen itself is absent)",
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "vertices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


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
    world_env = os.environ.get("WORLD_SIZE")
    if args.impl == "ours" and args.gpus > 1 and world_env is None:
        # `bench.py --gpus N` launches its own N ranks (one process per GPU)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    world = int(world_env or "1")
    if args.impl == "ours" and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
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
    out = (single_arm if cfg.get("single") else gpu_arm)(args, cfg, rank, world, local_rank)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
