"""Generate tests/golden/c4_doi.json (+ c4_doi_variant.json): the oracle's DOI chain
on the full C4 workload (1024^2 grid, 256 tiles of 64x64, c in [20, 400], band
1e-5 / 1e-4, binary weighting, z = 2, shift_scale = 1e-3).

Per tile: final c, DOI iterations, converged, doi_residual, residual_rms; per
step: (position, c the step ran with, residual, margin |r - eps|/eps against
the band edge the decision compared with).  The projections X^ = U U^T X of the
first tiles are not stored: past ~15 DOI steps the subspace itself is rounding-
dependent (below), so the fixture holds decisions and residuals only.

c4_doi_variant.json is the same chain through a second CPU restatement that
differs only in the solver (dense LU of L + delta I instead of the banded
Cholesky): DOI appends raw residual columns and re-applies R^2, which
amplifies rounding ~10x per step, so two correct implementations drift apart
(1e-9 relative after 10 steps, 1e-3 after 20, ~10% after 40).  The GPU test
bounds the GPU's distance from the oracle by this CPU-vs-CPU envelope.

The oracle is test infrastructure (oracle/specmesh_oracle.py restates
spectral.hpp:244-287 and pipeline.hpp:245-285).  Run from the repo root:
    python tests/golden/make_c4_doi.py              (oracle)
    python tests/golden/make_c4_doi.py --variant    (LU-solver restatement)
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

def margin(r, lo, hi):
    """distance of the decision to its nearest band edge, relative to that edge"""
    return min(abs(r - hi) / hi, abs(r - lo) / lo)


class LuOperator:
    """R^z by a dense LU of L + delta I (scipy lu_factor / lu_solve): the
    reference's operator up to rounding, through a different factorisation."""

    def __init__(self, lap, delta, z):
        import scipy.linalg as sla
        self.sla, self.z = sla, z
        self.lu = sla.lu_factor(lap.dense() + delta * np.eye(lap.size()))
        self.n = lap.size()

    def size(self):
        return self.n

    def apply(self, b):
        for _ in range(self.z):
            b = self.sla.lu_solve(self.lu, b)
        return b


def main(out_dir=os.path.dirname(os.path.abspath(__file__)), variant=False):
    w = synth.config("C4")
    subs = O.build_submeshes(w.mesh.adj_offsets, w.mesh.adj_cols, w.seg.members)
    cfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=w.c, c_min=w.c_min, c_max=w.c_max,
                           eps_low=w.eps_low, eps_high=w.eps_high, shift_scale=1e-3)
    trace = []
    t0 = time.time()

    def on_block(pos, sid, basis):
        if pos % 32 == 0:
            print(f"  position {pos}: c={basis.shape[1]} ({time.time() - t0:.0f} s)", flush=True)

    bb = O.compute_block_bases_doi(w.mesh.vertices, subs, w.seg.sequence, cfg, keep_bases=False, trace=trace,
                                   on_block=on_block, operator_factory=LuOperator if variant else None)
    tiles = []
    for sid in range(w.seg.count):
        st = bb.stats[sid]
        tiles.append(dict(c=st.subspace_size, iterations=st.oi_iterations, converged=bool(st.converged),
                          doi_residual=st.doi_residual, residual_rms=st.residual_rms))
    steps = [dict(pos=int(p), c=int(c), residual=float(r), margin=margin(r, w.eps_low, w.eps_high))
             for p, c, r in trace]
    doc = dict(config="C4", generator="tests/golden/make_c4_doi.py (oracle/specmesh_oracle.py)",
               solver="dense LU (variant)" if variant else "banded Cholesky (oracle)",
               eps_low=w.eps_low, eps_high=w.eps_high, c_min=w.c_min, c_max=w.c_max, shift_scale=1e-3,
               seconds=time.time() - t0, sequence=[int(s) for s in w.seg.sequence], tiles=tiles, steps=steps)
    name = "c4_doi_variant" if variant else "c4_doi"
    with open(os.path.join(out_dir, name + ".json"), "w") as f:
        json.dump(doc, f, indent=0)
    print(f"done in {time.time() - t0:.0f} s: {len(steps)} steps, c of tile 0 = {tiles[0]['c']}")


if __name__ == "__main__":
    main(variant="--variant" in sys.argv)
