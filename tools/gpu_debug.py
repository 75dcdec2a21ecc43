"""Quick GPU bring-up check of every primitive against the oracle (prints errors)."""
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import specmesh_oracle as O  # noqa: E402
import paper_1810_02719_b200 as G  # noqa: E402
from paper_1810_02719_b200 import synth  # noqa: E402


def step(name, fn):
    t = time.time()
    try:
        r = fn()
        print(f"[ok] {name} ({time.time()-t:.2f}s) {r if r is not None else ''}", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()


def main():
    ctx = G.Context(0)
    mesh = synth.small_grid(64, 64, 32, 32, seed=3, flip=5)
    seg = synth.grid_tiles(64, 64, 32, 32)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    lap0 = O.build_laplacian(subs[0], mesh.vertices, O.BINARY)
    state = {}

    def lap():
        rp, c, v, tr = G.build_laplacian(mesh, seg.members[0], "binary", ctx=ctx)
        assert np.array_equal(rp, lap0.rowptr) and np.array_equal(c, lap0.cols) and np.array_equal(v, lap0.vals)
        assert tr == lap0.trace()
        return f"nnz={c.size} trace={tr}"
    step("build_laplacian binary bit-exact", lap)

    delta = O.default_shift(lap0, 1e-3)
    op_o = O.ShiftedInverseOperator(lap0, delta, 2)

    def opc():
        state["op"] = G.ShiftedInverseOperator(lap0.rowptr, lap0.cols, lap0.vals, delta, 2, ctx=ctx)
    step("operator create", opc)
    rng = np.random.default_rng(0)
    B = rng.standard_normal((1024, 20))

    def app():
        y = state["op"].apply(B)
        yo = op_o.apply(B)
        return f"rel err {np.linalg.norm(y-yo)/np.linalg.norm(yo):.2e}"
    step("apply R^2", app)

    def app1():
        y = state["op"].apply_once(B)
        yo = op_o.apply_once(B)
        return f"rel err {np.linalg.norm(y-yo)/np.linalg.norm(yo):.2e}"
    step("apply_once", app1)

    def spmm():
        y = state["op"].spmm(B)
        A = lap0.to_scipy() + delta * np.eye(1024)
        yo = A @ B
        return f"rel err {np.linalg.norm(y-yo)/np.linalg.norm(yo):.2e}"
    step("spmm", spmm)

    def orth():
        q = G.orthonormalize(B, ctx=ctx)
        qo = O.orthonormalize(B)
        return f"max abs diff {np.abs(q-qo).max():.2e}  orth {np.abs(q.T@q-np.eye(20)).max():.2e}"
    step("orthonormalize", orth)

    def orth_rank():
        Bd = B.copy()
        Bd[:, 5] = Bd[:, 2]
        try:
            G.orthonormalize(Bd, ctx=ctx)
            return "NO ERROR (bad)"
        except G.SpecmeshError as e:
            try:
                O.orthonormalize(Bd)
            except O.Error as eo:
                return f"gpu: {e} | oracle: {eo}"
    step("orthonormalize rank deficient", orth_rank)

    w, V = O.dense_eigendecomposition(lap0)
    init = V[:, :40].copy()

    def oi():
        u = G.orthogonal_iteration(state["op"], init, 3)
        uo = O.orthogonal_iteration(op_o, init, 3)
        return f"angle {O.max_principal_angle(u, uo):.2e}  vs exact {O.max_principal_angle(u, init):.2e}"
    step("orthogonal_iteration", oi)

    def bottom():
        u, ev = G.bottom_subspace(state["op"], 40, return_eigenvalues=True)
        return f"angle {O.max_principal_angle(u, init):.2e} ev err {np.abs(ev - w[:40]).max():.2e}"
    step("bottom_subspace", bottom)

    X = subs[0].local_coords(mesh.vertices)

    def gi():
        cg = G.gft(init, X, ctx=ctx)
        co = O.gft(init, X)
        xh = G.igft(init, co, ctx=ctx)
        return f"gft {np.abs(cg-co).max():.2e} igft {np.abs(xh - O.igft(init, co)).max():.2e}"
    step("gft/igft", gi)

    def doi():
        r = G.dynamic_oi(state["op"], V[:, :20].copy(), X, 1e-3, 1e-2, 5, 200, 60)
        ro = O.dynamic_oi(op_o, V[:, :20].copy(), X, 1e-3, 1e-2, 5, 200, 60)
        ang = O.max_principal_angle(r.basis, ro.basis) if r.basis.shape == ro.basis.shape else -1
        return (f"gpu c={r.basis.shape[1]} t={r.iterations} res={r.residual:.6e} conv={r.converged} | "
                f"oracle c={ro.basis.shape[1]} t={ro.iterations} res={ro.residual:.6e} conv={ro.converged} ang={ang:.2e}")
    step("dynamic_oi", doi)

    cfg = G.PipelineConfig(weighting="binary", subspace_size=40, iterations=1, shift_scale=1e-3)
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=40, iterations=1, shift_scale=1e-3)

    def chain():
        bb = G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [40] * seg.count, want_bases=True, ctx=ctx)
        ob = O.compute_block_bases_fixed_sizes(mesh.vertices, subs, seg.sequence, ocfg, [40] * seg.count)
        angs = [O.max_principal_angle(bb.bases[i], ob.bases[i]) for i in range(seg.count)]
        rec = O.coarse_reconstruct_points(ob, mesh.vertices)
        rerr = np.abs(bb.reconstruction - rec).max() / np.abs(rec).max()
        rms = max(abs(bb.stats[i].residual_rms - ob.stats[i].residual_rms) for i in range(seg.count))
        return f"angles {max(angs):.2e} recon {rerr:.2e} rms diff {rms:.2e} timings {bb.timings}"
    step("chain fixed", chain)

    def chain_doi():
        cfgd = G.PipelineConfig(weighting="binary", basis_mode="doi", subspace_size=20, c_min=10, c_max=200,
                                eps_low=1e-3, eps_high=1e-2, shift_scale=1e-3)
        ocfgd = O.PipelineConfig(weighting=O.BINARY, subspace_size=20, c_min=10, c_max=200, eps_low=1e-3,
                                 eps_high=1e-2, shift_scale=1e-3)
        bb = G.compute_block_bases(mesh, seg, cfgd, want_bases=True, ctx=ctx)
        ob = O.compute_block_bases_doi(mesh.vertices, subs, seg.sequence, ocfgd)
        g = [(s.subspace_size, s.oi_iterations) for s in bb.stats]
        o = [(s.subspace_size, s.oi_iterations) for s in ob.stats]
        return f"gpu {g} oracle {o}"
    step("chain doi", chain_doi)


if __name__ == "__main__":
    main()
