"""Generate tests/golden/c4_doi.json + c4_doi_xhat.npz: the oracle's DOI chain
on the full C4 workload (1024^2 grid, 256 tiles of 64x64, c in [20, 400], band
1e-5 / 1e-4, binary weighting, z = 2, shift_scale = 1e-3).

Per tile: final c, DOI iterations, converged, doi_residual, residual_rms; per
step: (position, c the step ran with, residual, margin |r - eps|/eps against
the band edge the decision compared with).  The projections X^ = U U^T X of the
first tiles are a basis-invariant fingerprint of the tracked subspace.

The oracle is test infrastructure (oracle/specmesh_oracle.py restates
spectral.hpp:244-287 and pipeline.hpp:245-285).  Run from the repo root:
    python tests/golden/make_c4_doi.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import specmesh_oracle as O  # noqa: E402
from paper_1810_02719_b200 import synth  # noqa: E402

XHAT_TILES = 4


def margin(r, lo, hi):
    """distance of the decision to its nearest band edge, relative to that edge"""
    return min(abs(r - hi) / hi, abs(r - lo) / lo)


def main(out_dir=os.path.dirname(os.path.abspath(__file__))):
    w = synth.config("C4")
    subs = O.build_submeshes(w.mesh.adj_offsets, w.mesh.adj_cols, w.seg.members)
    cfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=w.c, c_min=w.c_min, c_max=w.c_max,
                           eps_low=w.eps_low, eps_high=w.eps_high, shift_scale=1e-3)
    trace, xhat = [], {}
    t0 = time.time()

    def on_block(pos, sid, basis):
        if pos < XHAT_TILES:
            x = subs[sid].local_coords(w.mesh.vertices)
            xhat[f"tile{sid}"] = basis @ (basis.T @ x)
        if pos % 32 == 0:
            print(f"  position {pos}: c={basis.shape[1]} ({time.time() - t0:.0f} s)", flush=True)

    bb = O.compute_block_bases_doi(w.mesh.vertices, subs, w.seg.sequence, cfg, keep_bases=False, trace=trace,
                                   on_block=on_block)
    tiles = []
    for sid in range(w.seg.count):
        st = bb.stats[sid]
        tiles.append(dict(c=st.subspace_size, iterations=st.oi_iterations, converged=bool(st.converged),
                          doi_residual=st.doi_residual, residual_rms=st.residual_rms))
    steps = [dict(pos=int(p), c=int(c), residual=float(r), margin=margin(r, w.eps_low, w.eps_high))
             for p, c, r in trace]
    doc = dict(config="C4", generator="tests/golden/make_c4_doi.py (oracle/specmesh_oracle.py)",
               eps_low=w.eps_low, eps_high=w.eps_high, c_min=w.c_min, c_max=w.c_max, shift_scale=1e-3,
               seconds=time.time() - t0, sequence=[int(s) for s in w.seg.sequence], tiles=tiles, steps=steps)
    with open(os.path.join(out_dir, "c4_doi.json"), "w") as f:
        json.dump(doc, f, indent=0)
    np.savez_compressed(os.path.join(out_dir, "c4_doi_xhat.npz"), **xhat)
    print(f"done in {time.time() - t0:.0f} s: {len(steps)} steps, c of tile 0 = {tiles[0]['c']}")


if __name__ == "__main__":
    main()
