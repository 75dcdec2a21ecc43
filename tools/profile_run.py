"""Small C5-shaped run for ncu captures: N chains of 512x512 grids (128 tiles of
32x64, c=200, t=1) through smg_run_chains, once (plus one warm-up)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1810_02719_b200 as G  # noqa: E402
from paper_1810_02719_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chains", type=int, default=8)
    ap.add_argument("--tiles", type=int, default=128)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    ctx = G.Context(0)
    base = synth.grid_mesh(512, 512, 5000, 0.01)
    seg = synth.grid_tiles(512, 512, 64, 32)
    seg = synth.Segmentation(seg.members[:a.tiles], np.arange(a.tiles, dtype=np.int32))
    meshes = []
    for i in range(a.chains):
        v = synth.grid_vertices(512, 512, 5000 + i, 0.01)
        meshes.append(synth.Mesh(v, base.faces, base.adj_offsets, base.adj_cols))
    cfg = G.PipelineConfig(weighting="binary", subspace_size=200, iterations=1, shift_scale=1e-3)
    for _ in range(a.reps):
        res = G.run_chains(meshes, [seg] * a.chains, cfg, [200] * a.tiles, want_recon=False, ctx=ctx)
    print("ok", res[0].timings)


if __name__ == "__main__":
    main()
