"""Dump the GPU's C4 DOI chain (per-tile outcome + per-step log) to
gpurun_out/c4_gpu.json for comparison with tests/golden/c4_doi*.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_02719_b200 as G  # noqa: E402
from paper_1810_02719_b200 import synth  # noqa: E402

w = synth.config("C4")
ctx = G.Context(0)
cfg = G.PipelineConfig(weighting="binary", basis_mode="doi", subspace_size=w.c, c_min=w.c_min, c_max=w.c_max,
                       eps_low=w.eps_low, eps_high=w.eps_high, shift_scale=1e-3)
ctx.doi_trace(True)
bb = G.compute_block_bases(w.mesh, w.seg, cfg, want_bases=False, ctx=ctx)
pos, cs, rs = ctx.read_doi_trace()
tiles = [dict(c=s.subspace_size, iterations=s.oi_iterations, converged=bool(s.converged), doi_residual=s.doi_residual,
              residual_rms=s.residual_rms) for s in bb.stats]
steps = [dict(pos=int(p), c=int(c), residual=float(r)) for p, c, r in zip(pos, cs, rs)]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(dict(tiles=tiles, steps=steps), open(os.path.join(ROOT, "gpurun_out", "c4_gpu.json"), "w"))
print("ok", len(steps))
