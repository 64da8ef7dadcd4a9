"""GPU: candidate selection fused into the int4 proxy kernel (fsel.cuh)
against the oracle's topk_select (linalg.hpp:157-176) + ascending sort
(hire.hpp:65-67) over the same integer proxy scores — bit-exact candidate
sets. Covers the fused path (rows > 8192, int8 x), its exact fallback
(bracket miss / list overflow on tied or degenerate score rows), batches
spanning several MMA n-tiles, zero-at-rest counters under CUDA-graph replay,
and equality with the unfused grid-wide selector (HIRE_FSEL=0)."""
import numpy as np
import pytest
import torch

from tests import _data

pytestmark = pytest.mark.gpu


def T(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dtype)


def N(t):
    return t.detach().cpu().numpy()


def _instance(H, O, V, d, seed, kind="lowrank"):
    if kind == "lowrank":
        w = _data.lowrank_plus_noise(V, d, 32, seed)
    elif kind == "int_ties":  # integer codes, unit scales: many exact score ties
        g = np.random.default_rng(seed)
        w = g.integers(-7, 8, size=(V, d)).astype(np.float32)
        w[:, 0] = 7.0  # absmax 7 on every row -> scale 1
    elif kind == "equal_rows":  # every row identical: every score ties
        g = np.random.default_rng(seed)
        w = np.tile(g.standard_normal((1, d)).astype(np.float32), (V, 1))
    else:
        raise ValueError(kind)
    codes, scales = O.quantize_int4(w)
    return w, H.ScoreMatrix(T(w)), H.ApproxScorer.quantized(codes, scales), codes, scales


def _want_cand(O, codes, scales, x, kp):
    s = O.q4_scores_int8(codes, scales, x, 0)
    idx, _, _ = O.topk_select(s, kp)
    return np.sort(idx.astype(np.uint32)), s


def _run(H, x, z, a, k, kp):
    return H.hire_topk(T(x), z, a, H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8))


@pytest.mark.parametrize("V,d,kp,B", [(8193, 128, 820, 1), (20000, 256, 1024, 3), (100000, 128, 1024, 8),
                                      (256000, 128, 1024, 1), (256000, 64, 2048, 2), (50000, 64, 1, 2),
                                      (60000, 64, 4000, 9), (40000, 64, 300, 17)])
def test_fused_candidates_bitexact(H, O, V, d, kp, B):
    w, z, a, codes, scales = _instance(H, O, V, d, V + kp)
    x = _data.queries(B, d, V)
    r = _run(H, x, z, a, 1, kp)
    for b in range(B):
        want, _ = _want_cand(O, codes, scales, x[b], kp)
        assert np.array_equal(N(r.cand[b]).astype(np.uint32), want), b


@pytest.mark.parametrize("kind", ["int_ties", "equal_rows"])
def test_fused_ties_and_fallback(H, O, kind):
    V, d, kp = 30000, 64, 700
    w, z, a, codes, scales = _instance(H, O, V, d, 4, kind)
    x = np.round(_data.queries(3, d, 5, scale=3.0)).astype(np.float32)
    x[2] = 0.0  # all-zero query: every score 0, ties broken by index
    r = _run(H, x, z, a, 1, kp)
    for b in range(3):
        want, _ = _want_cand(O, codes, scales, x[b], kp)
        assert np.array_equal(N(r.cand[b]).astype(np.uint32), want), b


def test_fused_equals_unfused(H, O, monkeypatch):
    V, d, kp, B = 120000, 128, 1024, 5
    w, z, a, codes, scales = _instance(H, O, V, d, 8)
    x = _data.queries(B, d, 9)
    r1 = _run(H, x, z, a, 64, kp)
    monkeypatch.setenv("HIRE_FSEL", "0")
    r0 = _run(H, x, z, a, 64, kp)
    assert torch.equal(r1.cand, r0.cand)
    assert torch.equal(r1.top_idx, r0.top_idx)
    assert torch.equal(r1.top_val, r0.top_val)


def test_fused_graph_replay(H, O):
    V, d, kp, B = 50000, 128, 512, 2
    w, z, a, codes, scales = _instance(H, O, V, d, 10)
    g = np.random.default_rng(11)
    xd = T(_data.queries(B, d, 12))
    cfg = H.HireConfig(k=8, k_prime=kp, x_mode=H.X_INT8)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        H.hire_topk(xd, z, a, cfg)  # workspace before capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            r = H.hire_topk(xd, z, a, cfg)
    for it in range(4):
        xh = (g.standard_normal((B, d)) / np.sqrt(d)).astype(np.float32)
        if it == 2:
            xh[1] = 0.0  # fallback inside a replay, then the fused path again
        xd.copy_(T(xh))
        graph.replay()
        torch.cuda.synchronize()
        for b in range(B):
            want, _ = _want_cand(O, codes, scales, xh[b], kp)
            assert np.array_equal(N(r.cand[b]).astype(np.uint32), want), (it, b)


def test_fused_topk_values_strict(H, O):
    # full hire_topk through the fused path, strict recompute: bit-exact
    V, d, k, kp = 40000, 256, 32, 512
    w, z, a, codes, scales = _instance(H, O, V, d, 13)
    x = _data.queries(2, d, 14)
    r = H.hire_topk(T(x), z, a, H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8, strict=True))
    for b in range(2):
        approx = O.q4_scores_int8(codes, scales, x[b], 0)
        o = O.hire_topk(w, x[b], approx, k, kp, 0)
        assert np.array_equal(N(r.cand[b]).astype(np.uint32), o["cand"])
        assert np.array_equal(N(r.top_idx[b]).astype(np.uint32), o["top_idx"])
        assert np.array_equal(N(r.top_val[b]).view(np.uint32), o["top_val"].view(np.uint32))


def test_fused_unordered_candidates_same_topk(H, O):
    # want_candidates=False: the fused selector emits candidates in any order;
    # the exact top-k (values, ties by index) must not change
    V, d, k, kp, B = 150000, 128, 64, 1024, 4
    w, z, a, codes, scales = _instance(H, O, V, d, 21)
    x = _data.queries(B, d, 22)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8)
    r1 = H.hire_topk(T(x), z, a, cfg)
    r0 = H.hire_topk(T(x), z, a, cfg, want_candidates=False)
    assert torch.equal(r1.top_idx, r0.top_idx)
    assert torch.equal(r1.top_val, r0.top_val)
    for b in range(B):
        want, _ = _want_cand(O, codes, scales, x[b], kp)
        assert np.array_equal(N(r1.cand[b]).astype(np.uint32), want)


def test_fused_post_kernel_equals_chain(H, O, monkeypatch):
    if not H.lib().hire_experiments_built():
        pytest.skip("experiments-build kernel (-DHIRE_EXPERIMENTS=1)")
    # opt-in single post-proxy launch (finisher + recompute + final top-k)
    V, d, k, kp, B = 60000, 256, 32, 512, 3
    w, z, a, codes, scales = _instance(H, O, V, d, 31)
    x = _data.queries(B, d, 32)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8)
    r0 = H.hire_topk(T(x), z, a, cfg)
    i0, p0 = H.softmax_topk(z, T(x), a, cfg)
    monkeypatch.setenv("HIRE_FSEL_POST", "1")
    for _ in range(2):
        r1 = H.hire_topk(T(x), z, a, cfg)
        i1, p1 = H.softmax_topk(z, T(x), a, cfg)
        assert torch.equal(r0.cand, r1.cand)
        assert torch.equal(r0.top_idx, r1.top_idx)
        assert torch.equal(r0.top_val, r1.top_val)
        assert torch.equal(i0, i1)
        torch.testing.assert_close(p0, p1, rtol=1e-6, atol=0)
