"""Per-config throughput of the single-chain configs C1-C4 (BASELINE.json),
one GPU, through the public Python API (host inputs, host outputs).

Prints one JSON line per config: vertices/s from the library's device-event
total (`timings["total"]`, laplacian -> stitched reconstruction) and from the
host wall clock around the call (H2D + D2H included), best of `--reps` after
one warm-up call.  C1-C3 are OI chains, C4 the dynamic-c chain.  The C5
batched config is bench.py's default workload.

  python tools/bench_configs.py [--configs C1,C2,C3,C4] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import paper_1810_02719_b200 as G
    from paper_1810_02719_b200 import synth
    ctx = G.Context(0)
    for name in args.configs.split(","):
        w = synth.config(name)
        if w.doi:
            cfg = G.PipelineConfig(weighting="binary", basis_mode="doi", subspace_size=w.c, c_min=w.c_min,
                                   c_max=w.c_max, eps_low=w.eps_low, eps_high=w.eps_high, shift_scale=1e-3)

            def run():
                return G.compute_block_bases(w.mesh, w.seg, cfg, ctx=ctx)
        else:
            cfg = G.PipelineConfig(weighting="binary", subspace_size=w.c, iterations=w.iterations, shift_scale=1e-3)

            def run():
                return G.compute_block_bases_fixed_sizes(w.mesh, w.seg, cfg, [w.c] * w.seg.count, ctx=ctx)
        run()
        import ctypes as C
        ctx.lib.smg_profile_enable(ctx.handle, 1)
        run()
        stages = {}
        for nm in ("assemble", "factor", "first_basis", "solve", "orthonormalize", "gram", "chol", "trmm", "project"):
            n_, t_ = C.c_int64(), C.c_double()
            ctx.lib.smg_profile_read(ctx.handle, nm.encode(), C.byref(n_), C.byref(t_))
            stages[nm] = {"launches": n_.value, "ms": round(t_.value, 3)}
        ctx.lib.smg_profile_enable(ctx.handle, 0)
        best_dev, best_wall, bb = 1e30, 1e30, None
        for _ in range(args.reps):
            t0 = time.perf_counter()
            bb = run()
            wall = time.perf_counter() - t0
            best_wall = min(best_wall, wall)
            best_dev = min(best_dev, bb.timings["total"])
        n = w.mesh.n
        sizes = [s.subspace_size for s in bb.stats]
        out = {"config": name, "vertices": n, "tiles": w.seg.count, "n_d": w.seg.block_size,
               "c": w.c if not w.doi else {"min": min(sizes), "max": max(sizes), "mean": sum(sizes) / len(sizes)},
               "device_s": best_dev, "wall_s": best_wall, "vertices_per_s_device": n / best_dev,
               "vertices_per_s_e2e": n / best_wall,
               "timings": {k: round(v, 6) for k, v in bb.timings.items()}, "stages_ms": stages}
        if w.doi:
            out["doi_steps"] = int(sum(s.oi_iterations for s in bb.stats))
            out["converged_blocks"] = int(sum(s.converged for s in bb.stats))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
