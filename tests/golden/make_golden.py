"""Per-function golden vectors from the REFERENCE implementation.

Run here (the container that has /root/reference), never on the GPU box:

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz (+ golden_payloads.npz): inputs and the
reference's outputs for every hot-path function at test-scale sizes,
plus reference-encoded entropy/tree payloads covering the parser's edge
cases.  The oracle (oracle/) and the CUDA path are both checked against it.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import hivc.bits as rbits  # noqa: E402
import hivc.entropy as rent  # noqa: E402
import hivc.flow as rflow  # noqa: E402
import hivc.homogeneous as rh  # noqa: E402
import hivc.pseudodiff as rp  # noqa: E402
import hivc.subdivision as rsub  # noqa: E402


def main():
    rng = np.random.default_rng(20081027)
    g = {}
    # ---- homogeneous inpainting (homogeneous.py:157-212)
    cases = [(12, 12, 0.1, 1e-6, 10000, True), (37, 53, 0.05, 1e-4, 160, False), (1, 40, 0.1, 1e-6, 10000, True),
             (17, 1, 0.2, 1e-6, 10000, True), (64, 96, 0.04, 1e-4, 160, False), (90, 160, 0.02, 1e-6, 10000, True),
             (8, 8, 1.0, 1e-6, 10000, True), (33, 65, 0.03, 1e-4, 3, False)]
    for i, (h, w, dens, tol, mi, strict) in enumerate(cases):
        f = rng.uniform(0, 255, (h, w))
        m = rng.uniform(size=(h, w)) < dens
        m.flat[rng.integers(h * w)] = True
        f = np.where(m, f, 0.0)
        st = {}
        u = rh.solve_homogeneous(f, m, tol=tol, max_iter=mi, strict=strict, stats=st)
        g[f"homog{i}_f"] = f
        g[f"homog{i}_m"] = m
        g[f"homog{i}_u"] = u
        g[f"homog{i}_cfg"] = np.array([tol, mi, strict], dtype=np.float64)
        g[f"homog{i}_iters"] = np.array(st["level_iterations"], dtype=np.int64)
        if h * w <= 64 * 64:
            g[f"homog{i}_dense"] = rh.solve_dense(f, m)
    # ---- block reconstruction / fit (pseudodiff.py:243-279)
    n = 300
    mc = np.zeros((n, 8, 8))
    masks = rng.uniform(size=(n, 8, 8)) < 0.08
    masks[np.arange(n), rng.integers(0, 8, n), rng.integers(0, 8, n)] = True
    mc[masks] = rng.normal(0, 60, masks.sum())
    a = rng.normal(0, 10, n)
    g["blocks_mc"] = mc
    g["blocks_a"] = a
    g["blocks_rec"] = rp.reconstruct_blocks(mc, a)
    g["blocks_eig"] = rp.greens_eigenvalues_harmonic()
    g["fscale2"] = rp._FSCALE2
    g["iscale2"] = rp._ISCALE2
    g["g8"] = rp._greens_block_matrix()
    fb = rng.normal(0, 8, (n, 8, 8))
    g["fit_f"] = fb
    g["fit_masks"] = masks
    ks = masks.reshape(n, 64).sum(1)
    cfull = np.zeros((n, 64))
    afit = np.zeros(n)
    for k in np.unique(ks):
        sel = np.flatnonzero(ks == k)
        c, aa = rp.solve_block_coefficients_batch(fb[sel], masks[sel])
        for j, i in enumerate(sel):
            cfull[i, masks[i].ravel()] = c[j]
        afit[sel] = aa
    g["fit_c"] = cfull.reshape(n, 8, 8)
    g["fit_a"] = afit
    # ---- warp (flow.py:94-127)
    h, w = 45, 70
    planes = [rng.uniform(0, 255, (h, w)), np.rint(rng.uniform(-255, 255, (h, w)))]
    u = rng.normal(0, 6, (h, w))
    v = rng.normal(0, 6, (h, w))
    u[0, :5] = [0.5, -0.5, 1e-9, 200.0, -300.0]
    v[1, :3] = [0.5, 1.5, -2.5]
    g["warp_planes"] = np.stack(planes)
    g["warp_u"] = u
    g["warp_v"] = v
    g["warp_out"] = np.stack(rflow.warp_planes(planes, u, v))
    # ---- Brox flow (flow.py:187-278), both pyramid factors of the configs
    sys.path.insert(0, str(HERE.parent.parent))
    from paper_2008_10273_b200.synth import synth_clip

    clip = synth_clip(2, 48, 64, blobs=4, rects=2, v=3.0, seed=5)[:, 0].astype(np.float64)
    g["brox_pair"] = clip
    for tag, sc in (("05", 0.5), ("095", 0.95)):
        ff = rflow.flow_brox(clip[1], clip[0], rflow.BroxParams(pyramid_scale=sc))
        g[f"brox{tag}_u"] = ff.u
        g[f"brox{tag}_v"] = ff.v
    np.savez_compressed(HERE / "golden.npz", **g)

    # ---- entropy + tree payloads (entropy.py, subdivision.py)
    p = {}
    sym_cases = [
        np.array([], dtype=np.int64),
        np.array([0]),
        np.array([3, 3, 3, 3]),
        rng.integers(0, 2, 50),
        rng.integers(0, 255, 5000),
        np.minimum(rng.geometric(0.3, 70000) - 1, 40),
    ]
    for i, s in enumerate(sym_cases):
        p[f"sym{i}_in"] = s
        p[f"sym{i}_payload"] = np.frombuffer(rent.encode_symbols(s), dtype=np.uint8)
    for tl in (5, 8, 12):
        s = rng.integers(0, 20, 300)
        p[f"symtl{tl}_in"] = s
        p[f"symtl{tl}_payload"] = np.frombuffer(rent.encode_symbols(s, table_log=tl), dtype=np.uint8)
    sv_cases = [
        np.array([], dtype=np.int64),
        np.array([0, 0, 0]),
        np.array([1, -1, 2, -2, 3, -3, 127, -127, 32767, -32767]),
        np.rint(rng.laplace(0, 20, 4000)).astype(np.int64),
    ]
    for i, s in enumerate(sv_cases):
        p[f"sv{i}_in"] = s
        p[f"sv{i}_payload"] = np.frombuffer(rent.encode_signed_values(s), dtype=np.uint8)
    for i, (h, w, pts) in enumerate([(1, 1, 1), (8, 8, 4), (5, 3, 7), (180, 320, 2304), (7, 8, 1)]):
        plane = rng.uniform(0, 255, (h, w))
        tree = rsub.subdivide_by_error(plane, pts)
        wr = rbits.BitWriter()
        rsub.serialize_tree(tree, wr)
        p[f"tree{i}_shape"] = np.array([h, w])
        p[f"tree{i}_bits"] = np.frombuffer(wr.getvalue(), dtype=np.uint8)
        p[f"tree{i}_nbits"] = np.array([len(wr)])
        p[f"tree{i}_leaves"] = np.array(tree.leaves(), dtype=np.int64).reshape(-1, 4)
        p[f"tree{i}_mask"] = rsub.mask_from_tree(tree)
    np.savez_compressed(HERE / "golden_payloads.npz", **p)
    print("wrote", HERE / "golden.npz", HERE / "golden_payloads.npz")


if __name__ == "__main__":
    main()
