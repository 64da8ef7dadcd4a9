"""GPU: the grid-wide candidate selector (select2.cuh) against the oracle's
topk_select (linalg.hpp:157-176) — bit-exact indices and values, ties by
ascending index, over sizes that hit every path (single-CTA small mode,
sampled pivots + window, window overflow / bracket-miss fallback) and
adversarial value distributions."""
import numpy as np
import pytest
import torch


pytestmark = pytest.mark.gpu


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def N(t):
    return t.cpu().numpy()


def _rows(n, seed):
    g = np.random.default_rng(seed)
    rows = {
        "normal": g.standard_normal(n),
        "int_ties": g.integers(-20, 20, size=n),
        "all_equal": np.zeros(n),
        "relu": np.maximum(g.standard_normal(n) - 2.0, 0.0),
        "ascending": np.sort(g.standard_normal(n)),
        "descending": -np.sort(g.standard_normal(n)),
        "spiky": np.where(g.random(n) < 0.001, 100.0 + g.random(n), g.random(n) * 1e-3),
        "two_level": np.where(np.arange(n) % 97 == 0, 1.0, 0.5),
    }
    return {k: v.astype(np.float32) for k, v in rows.items()}


def _check(H, O, v, k):
    idx, val, cl = H.topk_select(T(v), k)
    for b in range(v.shape[0]):
        wi, wv, wcl = O.topk_select(v[b], k)
        gi = N(idx[b]).astype(np.uint32)
        assert np.array_equal(gi, wi), (b, k, gi[:8], wi[:8])
        assert np.array_equal(N(val[b]).view(np.uint32), wv.view(np.uint32))
        assert cl == wcl


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 1000, 8191, 8192, 8193, 9000, 32768, 256000])
def test_select_distributions(H, O, n):
    rows = _rows(n, n)
    v = np.stack(list(rows.values()))
    ks = sorted({1, min(n, 7), max(1, n // 100), max(1, n // 8), max(1, n - 1), n})
    for k in [k for k in ks if k <= 16384]:  # ranked output: k <= kFinalMax
        _check(H, O, v, k)


@pytest.mark.parametrize("n,k", [(1_000_000, 2048), (1_000_000, 16384), (300_000, 9000)])
def test_select_large(H, O, n, k):
    g = np.random.default_rng(7)
    v = np.stack([g.standard_normal(n), np.maximum(g.standard_normal(n), 0.0)]).astype(np.float32)
    _check(H, O, v, k)


@pytest.mark.parametrize("n,kp", [(60000, 30000), (60000, 59999), (60000, 60000), (20000, 19000)])
def test_candidate_sets_large_k_prime(H, O, n, kp):
    # candidate sets (ascending indices) for k' near n go through hire_topk
    g = np.random.default_rng(n + kp)
    d, r = 16, 4
    z1 = g.standard_normal((r, d)).astype(np.float32)
    z2 = np.round(g.standard_normal((n, r)) * 2).astype(np.float32)  # integer proxy scores: ties
    w = g.standard_normal((n, d)).astype(np.float32)
    x = np.round(g.standard_normal((2, d))).astype(np.float32)
    a = H.ApproxScorer.low_rank(T(z1), T(z2))
    cfg = H.HireConfig(k=5, k_prime=kp, strict=True)
    res = H.hire_topk(T(x), H.ScoreMatrix(T(w)), a, cfg)
    for b in range(2):
        s = O.lowrank_scores(z1, z2, x[b], 0)
        want = O.hire_topk(w, x[b], s, 5, kp, 0)
        assert np.array_equal(N(res.cand[b]).astype(np.uint32), want["cand"])
        assert np.array_equal(N(res.top_idx[b]).astype(np.uint32), want["top_idx"])


def test_select_repeated_calls_reset_counters(H, O):
    # zero-at-rest counters: back-to-back calls with different shapes
    g = np.random.default_rng(3)
    for it in range(6):
        n = [50000, 9000, 256000, 20000, 256000, 8193][it]
        B = [1, 4, 2, 16, 1, 3][it]
        v = g.standard_normal((B, n)).astype(np.float32)
        _check(H, O, v, [1024, 100, 2048, 256, 1024, 8000][it])


def test_select_batch_many_queries(H, O):
    g = np.random.default_rng(5)
    v = g.standard_normal((64, 30000)).astype(np.float32)
    v[::3] = np.round(v[::3] * 4)  # ties on every third query
    _check(H, O, v, 300)


def test_select_in_cuda_graph(H, O):
    g = np.random.default_rng(9)
    v = T(g.standard_normal((2, 100000)).astype(np.float32))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        H.topk_select(v, 1000)  # workspace exists before capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            idx, val, _ = H.topk_select(v, 1000)
    for _ in range(3):
        v.copy_(T(g.standard_normal((2, 100000)).astype(np.float32)))
        graph.replay()
        torch.cuda.synchronize()
        h = N(v)
        for b in range(2):
            wi, wv, _ = O.topk_select(h[b], 1000)
            assert np.array_equal(N(idx[b]).astype(np.uint32), wi)


@pytest.mark.parametrize("n,kp", [(200000, 8000), (200000, 8192), (100000, 6000), (40000, 3000),
                                  (530000, 1024), (524288, 512)])
def test_list_path_candidates(H, O, n, kp):
    # the list-path selector (sampled lower bound -> staged per-CTA lists ->
    # finisher) near its limits: k' at the 8192-key list cap (the listed
    # count overflows -> exact fallback), integer proxy scores (ties), and
    # rows just above / at kFinMaxRows (2^19; above it the window chain runs)
    g = np.random.default_rng(n + kp)
    d, r = 16, 4
    z1 = g.standard_normal((r, d)).astype(np.float32)
    z2 = np.round(g.standard_normal((n, r)) * 2).astype(np.float32)
    w = g.standard_normal((n, d)).astype(np.float32)
    x = np.round(g.standard_normal((3, d))).astype(np.float32)
    a = H.ApproxScorer.low_rank(T(z1), T(z2))
    res = H.hire_topk(T(x), H.ScoreMatrix(T(w)), a, H.HireConfig(k=5, k_prime=kp, strict=True))
    for b in range(3):
        s = O.lowrank_scores(z1, z2, x[b], 0)
        want, _, _ = O.topk_select(s, kp)
        assert np.array_equal(N(res.cand[b]).astype(np.uint32), np.sort(want.astype(np.uint32))), b


@pytest.mark.parametrize("kind", ["spiky", "two_level", "relu", "ascending", "all_equal"])
def test_list_path_equals_window_chain(H, O, kind, monkeypatch):
    # same candidate sets from the list path and the window chain
    # (HIRE_SEL_NOLIST=1) on adversarial score rows through hire_topk
    n, kp, d = 150000, 2000, 8
    v = _rows(n, 5)[kind]
    z2 = v[:, None].astype(np.float32)  # rank-1 proxy: score_i = v_i * x
    z1 = np.zeros((1, d), np.float32)
    z1[0, 0] = 1.0
    x = np.zeros((2, d), np.float32)
    x[:, 0] = 1.0
    w = np.random.default_rng(6).standard_normal((n, d)).astype(np.float32)
    a = H.ApproxScorer.low_rank(T(z1), T(z2))
    cfg = H.HireConfig(k=4, k_prime=kp, strict=True)
    r1 = H.hire_topk(T(x), H.ScoreMatrix(T(w)), a, cfg)
    monkeypatch.setenv("HIRE_SEL_NOLIST", "1")
    r0 = H.hire_topk(T(x), H.ScoreMatrix(T(w)), a, cfg)
    assert torch.equal(r1.cand, r0.cand)
    assert torch.equal(r1.top_idx, r0.top_idx)
    want, _, _ = O.topk_select(v, kp)
    assert np.array_equal(N(r1.cand[0]).astype(np.uint32), np.sort(want.astype(np.uint32)))


@pytest.mark.parametrize("kp,k", [(33, 1), (64, 5), (100, 32), (1000, 33), (2048, 64), (700, 64)])
def test_final_topk_warp_sort_equals_range_select(H, O, monkeypatch, kp, k):
    # the ranked final top-k by per-warp register sorts + a merge tree
    # (final3_kernel, small batches) against the range-select kernel: same
    # indices, values and softmax, with duplicate rows (value ties broken by
    # index) and a pool padded past the candidates
    V, d, B = 4096, 64, 3
    g = np.random.default_rng(kp + k)
    w = g.standard_normal((V, d)).astype(np.float32)
    w[1::7] = w[0]  # many identical rows: exact-value ties
    x = g.standard_normal((B, d)).astype(np.float32)
    z = H.ScoreMatrix(T(w))
    a = H.ApproxScorer.quantize(z)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8, strict=True)
    monkeypatch.setenv("HIRE_FINAL3", "1")
    r1 = H.hire_topk(T(x), z, a, cfg)
    i1, p1 = H.softmax_topk(z, T(x), a, cfg)
    monkeypatch.setenv("HIRE_FINAL3", "0")
    r0 = H.hire_topk(T(x), z, a, cfg)
    i0, p0 = H.softmax_topk(z, T(x), a, cfg)
    assert torch.equal(r1.top_idx, r0.top_idx) and torch.equal(r1.top_val, r0.top_val)
    assert torch.equal(i1, i0)
    torch.testing.assert_close(p1, p0, rtol=1e-6, atol=0)
    codes, scales = a.export_q4()
    for b in range(B):
        o = O.hire_topk(w, x[b], O.q4_scores_int8(codes, scales, x[b], 0), k, kp, 0)
        assert np.array_equal(N(r1.top_idx[b]).astype(np.uint32), o["top_idx"])
        assert np.array_equal(N(r1.top_val[b]), o["top_val"])


@pytest.mark.parametrize("n", [4097, 8191, 8192])
@pytest.mark.parametrize("k", [1, 100, 820, 8000])
def test_small_row_histogram_select(H, O, monkeypatch, n, k):
    # sel_exact_fast_kernel (mid ranks over rows <= 8192, the FFN layers'
    # top-k' of 8192 units): forced for every rank, every distribution
    monkeypatch.setenv("HIRE_SEL_EXACT", "4")
    rows = _rows(n, 17)
    v = np.stack([rows[kind] for kind in sorted(rows)])
    _check(H, O, v, min(k, n))
