"""K2/K3 parity: co-occurrence counts are bit-exact with the reference."""

import hashlib

import numpy as np
import pytest

from conftest import golden
from paper_2511_19493_b200 import _lib
from paper_2511_19493_b200 import proximity as P

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["auto", "leaf", "leaf32", "tile"])
def pair_kernel(request, monkeypatch):
    """Every count test runs on both K3 kernels: the leaf-segmented walk of
    the K2 buckets (over 16-bit sample ids, and over the 32-bit perm), the
    compare tiles, and the default launch of both behind the device-side
    gate."""
    if request.param == "auto":
        monkeypatch.delenv("RFX_PAIRS_KERNEL", raising=False)
    else:
        monkeypatch.setenv("RFX_PAIRS_KERNEL", request.param[:4])
    monkeypatch.setenv("RFX_PAIRS_PERM16", "0" if request.param == "leaf32" else "1")
    return request.param


def brute(codes):
    n, B = codes.shape
    M = np.zeros((n, n))
    for b in range(B):
        c = codes[:, b]
        M += c[:, None] == c[None, :]
    return M / B


def test_random_fixtures_exact():
    # tests/test_proximity.py:74-87 and acceptance A5
    for seed in (0, 42):
        rng = np.random.default_rng(seed)
        for _ in range(20):
            n = int(rng.integers(5, 51))
            B = int(rng.integers(1, 21))
            codes = np.zeros((n, B), np.int32)
            lc = np.zeros(B, np.int32)
            for b in range(B):
                k = int(rng.integers(1, max(2, n // 2 + 1)))
                codes[:, b] = rng.integers(0, k, size=n)
                lc[b] = codes[:, b].max() + 1 + int(rng.integers(0, 2))  # may exceed max+1
            full = P.full_proximity(P.LeafMembership(codes, lc))
            assert np.array_equal(full.to_dense(), brute(codes))


def test_simple_pair_values():
    full = P.full_proximity(P.LeafMembership(np.array([[0], [0], [1]], np.int32),
                                             np.array([2], np.int32)))
    assert full.entry(0, 1) == 1.0 and full.entry(0, 2) == 0.0
    full2 = P.full_proximity(P.LeafMembership(np.array([[0, 0], [0, 1]], np.int32),
                                              np.array([2, 2], np.int32)))
    assert full2.entry(0, 1) == 0.5


def test_wine_counts_and_packed_bit_exact(wine50, wine_ds):
    g = golden("wine50.npz")
    mem = P.leaf_membership(wine50, wine_ds)
    full = P.full_proximity(mem)
    assert np.array_equal(full.packed, g["packed"])
    counts = P.pair_counts_device(mem, _lib.UPPER_I32).cpu().numpy()
    assert np.array_equal(counts.astype(np.int64), g["pair_counts"])


def test_synth2k_counts_sha(synth2k, fixtures):
    ds, forest = synth2k
    mem = P.leaf_membership(forest, ds)
    counts = P.pair_counts_device(mem, _lib.UPPER_I32).cpu().numpy()
    assert hashlib.sha256(counts.tobytes()).hexdigest() == fixtures["synth2k"]["counts_i32_sha"]


def test_row_block_layouts(orc):
    g = golden("synth2k.npz")
    codes, lc = g["codes"], g["leaf_counts"]
    mem = P.LeafMembership(codes, lc)
    n = codes.shape[0]
    full = P.pair_counts_device(mem, _lib.UPPER_I32).cpu().numpy()
    for lo, hi in [(0, 1), (5, 300), (1234, 1999), (1998, 2000), (700, 2000)]:
        blk = P.pair_counts_device(mem, _lib.BLOCK_I32, lo, hi).cpu().numpy().reshape(hi - lo, n)
        assert np.array_equal(blk, orc.block_counts(codes, lc, lo, hi))
        up = P.pair_counts_device(mem, _lib.UPPER_I32, lo, hi).cpu().numpy()
        s, e = P._row_start(n, lo), P._row_start(n, hi)
        assert np.array_equal(up, full[s:e])


def test_triblock_matches_reference(wine50, wine_ds):
    g = golden("wine50.npz")
    mem = P.leaf_membership(wine50, wine_ds)
    tb = P.triblock_proximity(mem, tau=0.05)
    assert np.array_equal(tb.dense.i, g["tb_dense_i"]) and np.array_equal(tb.dense.j, g["tb_dense_j"])
    assert np.array_equal(tb.dense.v, g["tb_dense_v"])
    assert np.array_equal(tb.sparse_i, g["tb_sparse_i"])
    assert np.array_equal(tb.sparse_j, g["tb_sparse_j"])
    assert np.array_equal(tb.sparse_v, g["tb_sparse_v"])
    assert all(v >= 0.05 for v in tb.dense.values())
    full = P.full_proximity(mem)
    tb2 = P.triblock_proximity(mem)  # default tau: every non-zero is dense (B < 1e4)
    assert tb2.sparse_count == 0
    assert np.array_equal(tb2.to_dense(), full.to_dense())


def test_triblock_all_one_leaf(wine_ds, built):
    from oracle.trainer import train
    from paper_2511_19493_b200.forest import TrainConfig
    f = train(wine_ds, TrainConfig(ntree=2, iseed=1, min_node_size=10**6))
    tb = P.triblock_proximity(P.leaf_membership(f, wine_ds), tau=0.5)
    n = wine_ds.n
    assert tb.dense_count == n * (n - 1) // 2 and tb.sparse_count == 0


def test_one_tree_row_sum_equals_leaf_size():
    codes = np.random.default_rng(4).integers(0, 6, size=(40, 1)).astype(np.int32)
    dense = P.full_proximity(P.LeafMembership(codes, np.array([6], np.int32))).to_dense()
    for i in range(40):
        assert dense[i].sum() == pytest.approx((codes[:, 0] == codes[i, 0]).sum())


def test_bucket_is_stable_counting_sort(synth2k):
    ds, forest = synth2k
    mem = P.leaf_membership(forest, ds)
    d = mem.device()
    perm, seg = d.buckets()
    perm, seg = perm.cpu().numpy(), seg.cpu().numpy()
    codes = golden("synth2k.npz")["codes"]
    n = codes.shape[0]
    first = (perm.view(np.uint32) >> 31).astype(bool)
    perm = perm & 0x7FFFFFFF
    for b in (0, 7, 39):
        want = np.argsort(codes[:, b], kind="stable")
        assert np.array_equal(perm[b], want)
        # RFXC_PERM_FIRST marks exactly the first member of every leaf
        sc = codes[want, b]
        assert np.array_equal(first[b], np.r_[True, sc[1:] != sc[:-1]])
        lo, hi = d.leaf_base_host[b], d.leaf_base_host[b + 1]
        starts = seg[lo:hi + 1] - b * n
        assert np.array_equal(np.diff(starts), np.bincount(codes[:, b], minlength=hi - lo))


def _bucket_case(codes, lc):
    from paper_2511_19493_b200.device import DeviceMembership
    d = DeviceMembership.from_host(codes, lc)
    perm, seg = d.buckets()
    return d, perm.cpu().numpy().view(np.uint32), seg.cpu().numpy()


@pytest.mark.parametrize("n,L,mode", [
    (1, 1, "dense"), (37, 3, "dense"), (4096, 200, "dense"), (4097, 256, "gaps"),
    (5000, 257, "dense"), (9000, 700, "gaps"), (20000, 40000, "gaps"),
    (70000, 70000, "sparse3"), (12000, 5000, "one_big"), (8193, 300, "tail_empty"),
])
def test_radix_bucket_edge_cases(built, n, L, mode):
    """K2 on hand-built memberships: one, two and three 8-bit passes
    (L <= 256, <= 65536, > 65536), partial tiles, leaves with no member at
    the start / middle / end of the code range, one leaf holding most samples.
    perm must be the stable argsort, RFXC_PERM_FIRST the leaf starts, seg the
    run starts (empty leaf = start of the next one), has_empty exact."""
    rng = np.random.default_rng(n + L)
    B = 3
    codes = np.empty((n, B), np.int32)
    for b in range(B):
        if mode == "dense":
            c = rng.integers(0, L, n)
            c[: min(n, L)] = np.arange(min(n, L))
        elif mode == "gaps":
            c = rng.integers(0, L, n) // 3 * 3 + (L > 3) * 1
            c = np.minimum(c, L - 1)
        elif mode == "sparse3":
            c = rng.integers(L - 300, L, n)
        elif mode == "one_big":
            c = np.where(rng.random(n) < 0.9, L // 2, rng.integers(0, L, n))
        else:  # tail_empty
            c = rng.integers(0, L - 40, n)
        codes[:, b] = c
    lc = np.full(B, L, np.int32)
    d, perm, seg = _bucket_case(codes, lc)
    any_empty = False
    for b in range(B):
        want = np.argsort(codes[:, b], kind="stable")
        assert np.array_equal(perm[b] & 0x7FFFFFFF, want)
        sc = codes[want, b]
        assert np.array_equal((perm[b] >> 31).astype(bool), np.r_[True, sc[1:] != sc[:-1]])
        cnt = np.bincount(codes[:, b], minlength=L)
        starts = seg[b * L:(b + 1) * L + 1] - b * n
        assert starts[0] == 0 and np.array_equal(np.diff(starts), cnt)
        any_empty |= bool((cnt == 0).any())
    assert seg[-1] == B * n
    assert bool(int(d.has_empty.item())) == any_empty


def test_bucket_tree_ranges_compose(synth2k):
    """rfxc_bucket_trees over [0, a) then [a, Bl) writes exactly what one call
    over [0, Bl) writes (perm, run starts, empty flag)."""
    import torch
    from paper_2511_19493_b200 import _lib
    ds, forest = synth2k
    d = P.leaf_membership(forest, ds).device()
    perm, seg = d.buckets()
    n, Bl = d.n, d.Bl
    p2 = torch.empty_like(perm)
    s2 = torch.empty_like(seg)
    he = torch.zeros(1, dtype=torch.int32, device=perm.device)
    lib = _lib.load()
    maxl = int(d.leaf_counts.max())
    for lo, hi in ((0, 13), (13, Bl)):
        scratch = torch.empty(int(lib.rfxc_bucket_scratch_bytes(n, hi - lo)), dtype=torch.uint8,
                              device=perm.device)
        _lib.call("rfxc_bucket_trees", _lib.ptr(d.codes_tm), n, Bl, _lib.ptr(d.leaf_base), maxl,
                  lo, hi, _lib.ptr(p2), _lib.ptr(s2), _lib.ptr(scratch), _lib.ptr(he),
                  _lib.stream_handle())
    assert torch.equal(p2, perm) and torch.equal(s2, seg)
    assert int(he.item()) == int(d.has_empty.item())


@pytest.mark.parametrize("window", ["2", "7", "64"])
def test_leaf_kernel_column_windows(orc, monkeypatch, window):
    """Rows wider than the shared-memory window are counted in several
    passes; narrow windows force many passes, runs longer than 32 members
    and members outside the window."""
    monkeypatch.setenv("RFX_PAIRS_KERNEL", "leaf")
    monkeypatch.setenv("RFXC_PAIRS_WINDOW", window)
    rng = np.random.default_rng(7)
    n, B = 300, 9
    codes = np.zeros((n, B), np.int32)
    lc = np.zeros(B, np.int32)
    for b in range(B):
        k = [1, 2, 3, 50, 299][b % 5]  # one-leaf trees: every pair shares a leaf
        codes[:, b] = rng.integers(0, k, size=n)
        lc[b] = k
    mem = P.LeafMembership(codes, lc)
    full = P.full_proximity(mem)
    assert np.array_equal(full.to_dense(), brute(codes))
    for lo, hi in [(0, 1), (17, 250), (298, 300)]:
        blk = P.pair_counts_device(mem, _lib.BLOCK_I32, lo, hi).cpu().numpy().reshape(hi - lo, n)
        assert np.array_equal(blk, orc.block_counts(codes, lc, lo, hi))


def test_kernel_choice_follows_leaf_sizes(monkeypatch):
    """Small leaves pick the leaf walk, one-leaf trees the compare tiles."""
    monkeypatch.delenv("RFX_PAIRS_KERNEL", raising=False)
    n, B = 1000, 4
    small = P.LeafMembership(np.tile(np.arange(n, dtype=np.int32)[:, None] % 400, (1, B)),
                             np.full(B, 400, np.int32))
    assert P.pair_kernel(small.device()) == "leaf"
    assert small.device().same_leaf_pairs() == B * (200 * 3 + 200 * 1)
    one = P.LeafMembership(np.zeros((n, B), np.int32), np.ones(B, np.int32))
    assert P.pair_kernel(one.device()) == "tile"
    assert one.device().same_leaf_pairs() == B * n * (n - 1) // 2


def test_device_gate_picks_the_tiles_for_one_leaf_trees(monkeypatch):
    """Default (gated) launch on trees whose leaves hold every sample: the
    gate selects the compare tiles, the leaf walk exits, counts are exact."""
    monkeypatch.delenv("RFX_PAIRS_KERNEL", raising=False)
    n, B = 700, 3
    codes = np.zeros((n, B), np.int32)
    mem = P.LeafMembership(codes, np.ones(B, np.int32))
    up = P.pair_counts_device(mem, _lib.UPPER_I32).cpu().numpy()
    assert int(mem.device().pair_gate().item()) == 0
    assert np.all(up == B)
