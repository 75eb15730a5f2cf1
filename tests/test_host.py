"""Host-side logic: planner, tier map, relayout, sharding, validation."""

import numpy as np
import pytest

from paper_2511_19493_b200 import distributed as D
from paper_2511_19493_b200 import proximity as P
from paper_2511_19493_b200.errors import BudgetError, DataError


def test_planner_golden_rows():
    # tests/test_proximity.py:280-321 / test_acceptance A4 of the reference
    plan = P.memory_plan(100_000, tree_count=10_000)
    assert plan["full_headline_bytes"] == 80_000_000_000
    assert plan["triblock_bytes"] / 2**30 == pytest.approx(29.8, rel=0.02)
    assert plan["lowrank_r32_bytes"]["i8"]["two_factor"] == 6_400_000
    assert plan["lowrank_r32_bytes"]["nf4"]["two_factor"] == 3_200_000
    assert plan["model"]["subtotal"] / 1e6 == pytest.approx(381.2, abs=0.1)
    assert P.memory_plan(1_000)["recommended"] == "full or triblock"
    assert P.memory_plan(50_000)["recommended"] == "triblock"
    assert P.memory_plan(100_000)["recommended"].startswith("lowrank")
    assert P.memory_plan(100_000, rank=32, mode="i8")["requested"]["bytes"]["two_factor"] \
        == 6_400_000


def test_budget_refusals_before_device_work():
    mem = P.LeafMembership(np.zeros((1000, 1), np.int32), np.array([1], np.int32))
    with pytest.raises(BudgetError) as e:
        P.full_proximity(mem, budget_bytes=1000)
    assert e.value.plan["samples"] == 1000
    with pytest.raises(DataError):
        P.triblock_proximity(mem, tau=1e-7)
    with pytest.raises(DataError):
        P.triblock_proximity(mem, tau=1.0)
    with pytest.raises(DataError):
        P.lowrank_proximity(mem, rank=0)
    with pytest.raises(DataError):
        P.lowrank_proximity(mem, rank=3, mode="q3")


def test_packed_index_is_triu_order():
    for n in (2, 3, 7, 20):
        e = 0
        for i in range(n):
            for j in range(i + 1, n):
                assert P.packed_index(n, i, j) == e
                e += 1


def test_pair_map_behaves_like_the_reference_dict():
    i = np.array([0, 0, 2], np.int32)
    j = np.array([1, 3, 3], np.int32)
    v = np.array([0.5, 0.25, 1.0])
    m = P.PairMap(4, i, j, v)
    assert len(m) == 3 and m[(0, 3)] == 0.25 and m.get((1, 2)) is None
    assert (2, 3) in m and (3, 2) not in m
    assert dict(m.items()) == {(0, 1): 0.5, (0, 3): 0.25, (2, 3): 1.0}
    assert set(m) == {(0, 1), (0, 3), (2, 3)} and sorted(m.values()) == [0.25, 0.5, 1.0]
    tb = P.TriBlock(4, 2, 0.3, m, np.array([1], np.int32), np.array([2], np.int32),
                    np.array([0.1]))
    assert tb.entry(3, 2) == 1.0 and tb.entry(1, 2) == 0.1 and tb.entry(1, 3) == 0.0
    assert tb.entry(1, 1) == 1.0 and tb.stored_pairs == 4
    dense = tb.to_dense()
    assert dense[3, 0] == 0.25 and dense[2, 1] == 0.1


def test_full_triangle_accessors():
    ft = P.FullTriangle(n=3, tree_count=2, packed=np.array([0.5, 0.0, 1.0]))
    assert ft.entry(2, 1) == 1.0 and ft.entry(0, 0) == 1.0
    with pytest.raises(IndexError):
        ft.entry(0, 3)
    assert ft.to_dense()[1, 0] == 0.5


def host_pack(trees, p, col_cat, layout):
    """Call the C++ host packer (rfxc_forest_pack_host) — no GPU needed."""
    import ctypes
    from paper_2511_19493_b200 import _lib
    B = len(trees)
    keep, tabs = [], []
    for name, dt in (("status", np.int8), ("split_var", np.int32), ("threshold", np.float64),
                     ("cat_mask", np.int64), ("left", np.int32), ("right", np.int32)):
        arrs = [np.ascontiguousarray(getattr(t, name), dtype=dt) for t in trees]
        keep += arrs
        tabs.append(np.array([a.ctypes.data for a in arrs], dtype=np.uintp))
    counts = np.array([len(t.status) for t in trees], dtype=np.int64)
    rec = 16 if layout == _lib.NODES_F64 else 8
    off = np.empty(B + 1, np.int64)
    lc = np.empty(B, np.int32)
    cc = np.ascontiguousarray(col_cat, dtype=np.uint8)
    P = ctypes.c_void_p

    def call(dst):
        _lib.call("rfxc_forest_pack_host", *(t.ctypes.data_as(P) for t in tabs),
                  counts.ctypes.data_as(P), B, cc.ctypes.data_as(P), p, layout,
                  dst, off.ctypes.data_as(P), lc.ctypes.data_as(P), 2)
    nrec = int(counts.sum())
    if layout == _lib.NODES_F32_B2:  # sizing call first
        call(None)
        nrec = int(off[B])
    out = np.zeros(nrec * rec, dtype=np.uint8)
    call(out.ctypes.data_as(P))
    return out, off, lc


def walk_f32(rec, off, b, x, p):
    """Decode the 8-byte records and descend (mirror of traverse_kernel)."""
    from paper_2511_19493_b200.device import feature_bits
    fb = feature_bits(p)
    words = rec.view(np.uint32).reshape(-1, 2)
    node = 0
    while True:
        w0, w1 = int(words[off[b] + node, 0]), int(words[off[b] + node, 1])
        if w1 == 0:
            return w0
        f, cat, left = w1 & ((1 << fb) - 1), (w1 >> fb) & 1, w1 >> (fb + 1)
        v = np.float32(x[f])
        if cat:
            go = ((w0 >> int(v)) & 1) == 1 if int(v) < 32 else False
        else:
            go = v <= np.uint32(w0).view(np.float32)
        node = left + (0 if go else 1)


def walk_b2(rec, off, b, x, p):
    """Decode the 32-byte two-level groups and descend two levels per group
    fetch (mirror of traverse_kernel's B2 path)."""
    from paper_2511_19493_b200.device import feature_bits
    fb = feature_bits(p)
    words = rec.view(np.uint32).reshape(-1, 2)
    o = int(off[b])

    def decide(w0, w1):
        f, cat = w1 & ((1 << fb) - 1), (w1 >> fb) & 1
        v = np.float32(x[f])
        if cat:
            return ((w0 >> int(v)) & 1) == 1 if int(v) < 32 else False
        return v <= np.uint32(w0).view(np.float32)

    w0, w1 = int(words[o, 0]), int(words[o, 1])
    while True:
        if w1 == 0:
            return w0
        go = decide(w0, w1)
        rint = (w1 >> (fb + 1)) & 1
        g = o + (w1 >> (fb + 2)) + (4 if (not go and rint) else 0)
        assert (g - o) % 4 == 0  # 32-byte groups
        a = words[g:g + 4]
        y = a[0] if (go or rint) else a[1]
        if int(y[1]) == 0:
            return int(y[0])
        n2 = a[2] if decide(int(y[0]), int(y[1])) else a[3]
        w0, w1 = int(n2[0]), int(n2[1])


def test_host_packer_b2_layout(orc, mixed):
    """Two-level group layout: same leaf codes as the reference on a trained
    mixed (categorical) forest and on the hand-built tree with right != left+1
    (plus a single-leaf tree); trees and groups 32-byte aligned."""
    from conftest import golden
    from paper_2511_19493_b200 import _lib
    ds, forest = mixed
    X = ds.values.astype(np.float32).astype(np.float64)
    codes, lc_ref = orc.leaf_membership(forest.trees, forest.col_cat, X)
    rec, off, lc = host_pack(forest.trees, ds.p, forest.col_cat, _lib.NODES_F32_B2)
    assert np.array_equal(lc, lc_ref)
    assert np.all(off % 4 == 0) and np.all(np.diff(off) >= [len(t.status) for t in forest.trees])
    for i in range(0, ds.n, 5):
        for b in range(0, forest.ntree, 2):
            assert walk_b2(rec, off, b, X[i], ds.p) == codes[i, b]

    class T:
        pass
    h = golden("handbuilt.npz")
    t = T()
    t.status, t.split_var, t.threshold = h["status"], h["split_var"], h["threshold"]
    t.cat_mask, t.left, t.right = np.zeros(7, np.int64), h["left"], h["right"]
    stump = T()  # a single-leaf tree
    stump.status, stump.split_var, stump.threshold = np.array([1], np.int8), np.zeros(1), np.zeros(1)
    stump.cat_mask, stump.left, stump.right = np.zeros(1, np.int64), np.zeros(1), np.zeros(1)
    rec, off, lc = host_pack([t, stump], 2, np.zeros(2), _lib.NODES_F32_B2)
    assert list(lc) == [4, 1]
    for x, want in zip(h["points"], h["codes"]):
        assert walk_b2(rec, off, 0, x, 2) == want
        assert walk_b2(rec, off, 1, x, 2) == 0


def _random_tree(rng, n_internal, p, caterpillar=False):
    """Breadth-first numbered binary tree (siblings adjacent) of random shape;
    caterpillar=True: every right child is a leaf (depth = n_internal)."""
    class T:
        pass
    status, left = [0], [0]
    frontier = [0]
    made = 1
    while made < n_internal:
        x = frontier.pop(rng.integers(len(frontier)) if not caterpillar else 0)
        left[x] = len(status)
        for c in range(2):
            status.append(1)
            left.append(0)
        for c, ch in enumerate((left[x], left[x] + 1)):
            if made < n_internal and (c == 0 if caterpillar else rng.random() < 0.9):
                status[ch] = 0
                frontier.append(ch)
                made += 1
        if not frontier:
            break
    for x in frontier:  # unexpanded internal nodes become leaves
        status[x] = 1
    # renumber breadth-first (siblings adjacent) from the root
    nodes, q = [0], 0
    while q < len(nodes):
        x = nodes[q]
        q += 1
        if status[x] == 0:
            nodes += [left[x], left[x] + 1]
    new = {o: i for i, o in enumerate(nodes)}
    t = T()
    m = len(nodes)
    t.status = np.array([status[o] for o in nodes], np.int8)
    t.left = np.array([new[left[o]] if status[o] == 0 else 0 for o in nodes], np.int32)
    t.right = np.where(t.status == 0, t.left + 1, 0).astype(np.int32)
    t.split_var = rng.integers(0, p, m).astype(np.int32)
    t.threshold = rng.normal(size=m)
    t.cat_mask = np.zeros(m, np.int64)
    return t


@pytest.mark.parametrize("shape", ["random", "caterpillar"])
def test_host_packer_b2_random_shapes(built, shape):
    """Random and maximally unbalanced trees: the two-level groups route every
    point like the reference node order."""
    from paper_2511_19493_b200 import _lib
    rng = np.random.default_rng(11 if shape == "random" else 12)
    p = 5
    trees = [_random_tree(rng, int(k), p, caterpillar=(shape == "caterpillar"))
             for k in rng.integers(1, 300, size=6)]
    r1, o1, l1 = host_pack(trees, p, np.zeros(p), _lib.NODES_F32)
    r2, o2, l2 = host_pack(trees, p, np.zeros(p), _lib.NODES_F32_B2)
    assert np.array_equal(l1, l2)
    pts = rng.normal(size=(200, p)).astype(np.float32).astype(np.float64)
    for b in range(len(trees)):
        for x in pts:
            assert walk_b2(r2, o2, b, x, p) == walk_f32(r1, o1, b, x, p)


def test_host_packer_relayout_keeps_codes(built):
    """Hand-built tree with right != left + 1 (tests/test_forest.py:170-185):
    relaid out breadth-first by the C++ packer, leaf ordinals preserved."""
    from conftest import golden
    from paper_2511_19493_b200 import _lib

    class T:
        pass
    h = golden("handbuilt.npz")
    t = T()
    t.status, t.split_var, t.threshold = h["status"], h["split_var"], h["threshold"]
    t.cat_mask, t.left, t.right = np.zeros(7, np.int64), h["left"], h["right"]
    rec, off, lc = host_pack([t], 2, np.zeros(2), _lib.NODES_F32)
    assert lc[0] == 4
    for x, want in zip(h["points"], h["codes"]):
        assert walk_f32(rec, off, 0, x, 2) == want


def test_host_packer_matches_oracle_on_trained_forest(orc, mixed):
    """8-byte records + round-down thresholds route every sample like the
    reference (categorical masks included) when the values are f32-exact."""
    from paper_2511_19493_b200 import _lib
    ds, forest = mixed
    X = ds.values.astype(np.float32).astype(np.float64)  # make f32-exact copy
    codes, lc_ref = orc.leaf_membership(forest.trees, forest.col_cat, X)
    rec, off, lc = host_pack(forest.trees, ds.p, forest.col_cat, _lib.NODES_F32)
    assert np.array_equal(lc, lc_ref)
    for i in range(0, ds.n, 7):
        for b in range(0, forest.ntree, 3):
            assert walk_f32(rec, off, b, X[i], ds.p) == codes[i, b]


def test_values_to_f32_host_exactness(built):
    import ctypes
    from paper_2511_19493_b200 import _lib
    P = ctypes.c_void_p
    for vals, want in ((np.array([1.5, -2.25, 3.0]), 1), (np.array([0.1, 1.0]), 0)):
        out = np.empty(len(vals), np.float32)
        ex = np.zeros(1, np.int32)
        _lib.call("rfxc_values_to_f32_host", vals.ctypes.data_as(P), len(vals),
                  out.ctypes.data_as(P), ex.ctypes.data_as(P), 2)
        assert ex[0] == want and np.array_equal(out, vals.astype(np.float32))


def test_tree_and_row_shards_cover_exactly():
    for B, w in [(500, 8), (7, 3), (1000, 4)]:
        s = [D.tree_shard(B, r, w) for r in range(w)]
        assert s[0][0] == 0 and s[-1][1] == B
        assert all(a[1] == b[0] for a, b in zip(s, s[1:]))
        assert max(h - l for l, h in s) - min(h - l for l, h in s) <= 1
    for n, w in [(50_000, 8), (10, 3), (200_000, 2)]:
        s = [D.row_shard(n, r, w) for r in range(w)]
        assert s[0][0] == 0 and s[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(s, s[1:]))
        area = [P._row_start(n, h) - P._row_start(n, l) for l, h in s]
        if n > 1000:
            assert max(area) / min(area) < 1.01


def test_leafmembership_mirrors_reference_dataclass():
    codes = np.array([[0, 1], [0, 0], [1, 1]], np.int32)
    mem = P.LeafMembership(codes=codes, leaf_counts=np.array([2, 2], np.int32))
    assert mem.n == 3 and mem.tree_count == 2 and mem.total_leaves == 4
    M = mem.onehot()
    brute = sum((codes[:, b][:, None] == codes[:, b][None, :]) for b in range(2)) / 2
    assert np.allclose((M @ M.T).toarray(), brute, atol=1e-12)


def test_product_path_has_no_cpu_fallback(monkeypatch):
    """Without a CUDA device the product raises instead of computing on CPU."""
    import torch
    from paper_2511_19493_b200.errors import RfxError
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    mem = P.LeafMembership(np.zeros((10, 2), np.int32), np.array([1, 1], np.int32))
    with pytest.raises(RfxError):
        P.full_proximity(mem)
    with pytest.raises(RfxError):
        P.lowrank_proximity(mem, rank=2)
