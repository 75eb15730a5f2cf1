"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py            # small fixtures (~1 min)
    python tests/golden/make_golden.py --scale    # 10k / 50k checksums (~10 min)

The reference package is imported read-only from /root/reference/pkg/src.
Nothing here runs on the GPU box; the tests only read the committed files.
"""

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import rfx  # noqa: E402
from rfx import mds as rmds  # noqa: E402
from rfx import proximity as rprox  # noqa: E402
from rfx.forest import forest_to_bytes  # noqa: E402
from rfx.rng import Pcg32  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    if isinstance(a, bytes):
        return hashlib.sha256(a).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_synthetic(n, p, C=4, seed=0, p_inf=None, sep=1.0):
    """SURVEY §8(d) generator (restated in paper_2511_19493_b200.dataset)."""
    p_inf = min(p, 10) if p_inf is None else p_inf
    rng = np.random.default_rng(seed)
    y = rng.integers(0, C, n)
    centers = rng.normal(0, sep, (C, p_inf))
    X = rng.standard_normal((n, p)).astype(np.float32)
    X[:, :p_inf] += centers[y].astype(np.float32)
    return X.astype(np.float64), y


def pcg_kats():
    out = []
    for seed, seq in [(0, 0), (-5, 1), (7, 3), (123, 4), (2**40 + 3, 5), (17, 7)]:
        g = Pcg32(seed, seq)
        u32 = [g.next_u32() for _ in range(8)]
        bnd = [g.bounded(b) for b in (1, 2, 3, 1000, 178, 100000, 2**31 + 11)]
        nrm = Pcg32(seed, seq).normals(9)
        out.append(dict(seed=seed, seq=seq, u32=u32, bounded=bnd,
                        normals=[float(x).hex() for x in nrm]))
    return out


def pmax_draw_kats():
    """The 2048 bounded draws of the pmax pair sampler, Pcg32(seed, 4)
    (proximity.py:409-417), for a few (seed, n)."""
    out = []
    for seed, n in [(0, 178), (5, 2000), (0, 100_000), (-3, 2**31 + 11), (7, 3)]:
        g = Pcg32(seed, 4)
        out.append(dict(seed=seed, n=n, draws=[int(g.bounded(n)) for _ in range(2048)]))
    return out


def lowrank_record(mem, rank, mode, seed):
    lr = rprox.lowrank_proximity(mem, rank=rank, mode=mode, seed=seed)
    rec = dict(rank=lr.rank, degraded=lr.rank_degraded, pmax=lr.pmax,
               data=lr.factor.data, scales=lr.factor.scales if lr.factor.scales is not None
               else np.empty(0))
    return lr, rec


def small():
    from sklearn.datasets import load_wine
    w = load_wine()
    fx = {}
    # --- Wine, B=50, iseed=17 -------------------------------------------------
    ds = rfx.from_arrays(w.data, w.target)
    f = rfx.train(ds, rfx.TrainConfig(ntree=50, iseed=17))
    mem = rprox.leaf_membership(f, ds)
    full = rprox.full_proximity(mem)
    counts = rprox._pair_counts(mem)
    lr, rec = lowrank_record(mem, 16, "i8", 5)
    emb = rmds.mds_lowrank(lr, rmds.PowerIterConfig(seed=0))
    efull = rmds.mds_full(full)
    tb = rprox.triblock_proximity(mem, tau=0.05)
    dk = sorted(tb.dense)
    lrf, recf = lowrank_record(mem, 32, "f32", 0)
    v = np.random.default_rng(3).normal(size=ds.n)
    gmv = rmds.gram_matvec(lr, v)
    np.savez_compressed(
        os.path.join(HERE, "wine50.npz"), codes=mem.codes, leaf_counts=mem.leaf_counts,
        pair_counts=counts, packed=full.packed,
        lr_data=rec["data"], lr_scales=rec["scales"], lr_pmax=rec["pmax"],
        lrf_data=recf["data"], lrf_pmax=recf["pmax"],
        mds_coords=emb.coordinates, mds_eig=emb.eigenvalues, mds_iter=emb.iterations,
        mds_resid=emb.residuals, mds_conv=emb.converged,
        mdsfull_coords=efull.coordinates, mdsfull_eig=efull.eigenvalues,
        tb_dense_i=np.array([k[0] for k in dk], np.int32),
        tb_dense_j=np.array([k[1] for k in dk], np.int32),
        tb_dense_v=np.array([tb.dense[k] for k in dk]), tb_sparse_i=tb.sparse_i,
        tb_sparse_j=tb.sparse_j, tb_sparse_v=tb.sparse_v, gmv_v=v, gmv_w=gmv)
    fx["wine50"] = dict(rfx1_sha=sha(forest_to_bytes(f)), ntree=50, iseed=17)
    # --- Wine single-node trees (tests/test_proximity.py:33-37) -------------
    f1 = rfx.train(ds, rfx.TrainConfig(ntree=3, iseed=1, min_node_size=10**6))
    fx["wine_stumps"] = dict(rfx1_sha=sha(forest_to_bytes(f1)))
    # --- synthetic 2000 x 20, B = 40 --------------------------------------------
    X, y = make_synthetic(2000, 20, seed=1)
    ds2 = rfx.from_arrays(X, y)
    f2 = rfx.train(ds2, rfx.TrainConfig(ntree=40, iseed=1))
    mem2 = rprox.leaf_membership(f2, ds2)
    c2 = rprox._pair_counts(mem2)
    lr2, rec2 = lowrank_record(mem2, 32, "i8", 0)
    emb2 = rmds.mds_lowrank(lr2, rmds.PowerIterConfig(seed=0))
    np.savez_compressed(
        os.path.join(HERE, "synth2k.npz"), codes=mem2.codes, leaf_counts=mem2.leaf_counts,
        lr_data=rec2["data"], lr_scales=rec2["scales"], lr_pmax=rec2["pmax"],
        mds_coords=emb2.coordinates, mds_eig=emb2.eigenvalues, mds_iter=emb2.iterations)
    fx["synth2k"] = dict(rfx1_sha=sha(forest_to_bytes(f2)), counts_i32_sha=sha(
        c2.astype(np.int32)), counts_sum=int(c2.sum()), n=2000, p=20, ntree=40, iseed=1,
        data_seed=1)
    # --- mixed categorical columns ------------------------------------------------
    rng = np.random.default_rng(5)
    Xc = np.column_stack([rng.integers(0, 5, 300), rng.normal(size=300),
                          rng.integers(0, 3, 300), rng.normal(size=300)]).astype(float)
    yc = ((Xc[:, 0] % 2) + (Xc[:, 1] > 0) + (Xc[:, 2] == 1)).astype(int)
    cols = (rfx.ColumnKind("categorical", tuple("abcde")), rfx.ColumnKind("numeric"),
            rfx.ColumnKind("categorical", ("x", "y", "z")), rfx.ColumnKind("numeric"))
    dsc = rfx.from_arrays(Xc, yc, columns=cols)
    fc = rfx.train(dsc, rfx.TrainConfig(ntree=12, iseed=4))
    memc = rprox.leaf_membership(fc, dsc)
    np.savez_compressed(os.path.join(HERE, "mixed.npz"), X=Xc, y=yc, codes=memc.codes,
                        leaf_counts=memc.leaf_counts)
    fx["mixed"] = dict(rfx1_sha=sha(forest_to_bytes(fc)), ntree=12, iseed=4)
    # --- hand-built tree with right != left + 1 (tests/test_forest.py:170-185) ---
    status = np.array([0, 0, 1, 0, 1, 1, 1], np.int8)
    split_var = np.array([0, 1, -1, 0, -1, -1, -1], np.int32)
    threshold = np.array([0.5, 0.25, 0.0, 0.75, 0, 0, 0], np.float64)
    left = np.array([3, 4, -1, 6, -1, -1, -1], np.int32)
    right = np.array([1, 2, -1, 5, -1, -1, -1], np.int32)
    zeros = np.zeros(7, np.int32)
    tree = rfx.Tree(status, split_var, threshold, np.zeros(7, np.int64), left, right, zeros,
                    np.zeros((7, 2), np.int64), zeros, np.zeros(7, np.int64),
                    np.zeros(2, np.uint8))
    pts = np.random.default_rng(8).uniform(0, 1, size=(64, 2))
    pts[:4] = [[0.5, 0.25], [0.75, 0.1], [0.5, 0.9], [0.76, 0.25]]  # x == tau boundaries
    hb = tree.leaf_codes()[rfx.classify_all(tree, np.asfortranarray(pts))]
    np.savez_compressed(os.path.join(HERE, "handbuilt.npz"), status=status,
                        split_var=split_var, threshold=threshold, left=left, right=right,
                        points=pts, codes=hb)
    with open(os.path.join(HERE, "pcg32.json"), "w") as fh:
        json.dump(pcg_kats(), fh, indent=1)
    with open(os.path.join(HERE, "pcg32_pmax.json"), "w") as fh:
        json.dump(pmax_draw_kats(), fh)
    with open(os.path.join(HERE, "fixtures.json"), "w") as fh:
        json.dump(fx, fh, indent=1, sort_keys=True)


def scale(only=None):
    path = os.path.join(HERE, "scale.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name, n, p, B, do_counts, do_lr in [("10k", 10_000, 50, 500, True, True),
                                             ("50k", 50_000, 100, 500, True, False),
                                             ("100k", 100_000, 100, 500, False, True)]:
        if only and name not in only:
            continue
        t0 = time.time()
        X, y = make_synthetic(n, p, seed=0)
        ds = rfx.from_arrays(X, y)
        f = rfx.train(ds, rfx.TrainConfig(ntree=B, iseed=1))
        mem = rprox.leaf_membership(f, ds)
        rec = dict(n=n, p=p, ntree=B, iseed=1, data_seed=0,
                   rfx1_sha=sha(forest_to_bytes(f)), codes_sha=sha(mem.codes),
                   total_leaves=int(mem.leaf_counts.sum()))
        if do_counts:
            c = rprox._pair_counts(mem)
            rec["counts_i32_sha"] = sha(c.astype(np.int32))
            rec["counts_sum"] = int(c.sum())
            rec["counts_nonzero"] = int(np.count_nonzero(c))
            del c
        if do_lr:
            lr = rprox.lowrank_proximity(mem, rank=32, mode="i8", seed=0)
            emb = rmds.mds_lowrank(lr, rmds.PowerIterConfig(seed=0))
            np.savez_compressed(os.path.join(HERE, f"lowrank_{name}.npz"), data=lr.factor.data,
                                scales=lr.factor.scales, pmax=lr.pmax,
                                mds_coords=emb.coordinates, mds_eig=emb.eigenvalues,
                                mds_iter=np.asarray(emb.iterations))
        rec["seconds"] = time.time() - t0
        out[name] = rec
        print(name, rec, flush=True)
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", action="store_true")
    ap.add_argument("--only", nargs="*", help="scale configs to (re)generate, e.g. 100k")
    ap.add_argument("--pmax-kats", action="store_true", help="only tests/golden/pcg32_pmax.json")
    a = ap.parse_args()
    if a.pmax_kats:
        with open(os.path.join(HERE, "pcg32_pmax.json"), "w") as fh:
            json.dump(pmax_draw_kats(), fh)
    else:
        scale(a.only) if a.scale else small()
