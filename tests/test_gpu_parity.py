"""Parity of the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  * integer work (int4 x int8 -> int32 proxy scores, candidate sets, the
    K9 proxy build, selection over identical values): bit-exact;
  * strict mode (sequential fp32, no contraction): bit-exact with the
    reference's own arithmetic, hence identical index sets and values;
  * fast mode fp paths: values within 1e-5 relative (fp32) / 1e-3 (bf16),
    index sets identical except at near-ties |dscore| <= 1e-5 relative.
"""
import numpy as np
import pytest
import torch

from tests import _data

pytestmark = pytest.mark.gpu

DEV = "cuda"


def T(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV).to(dtype)


def N(t):
    return t.detach().cpu().numpy()


def assert_sets_near_tie(got_idx, want_idx, scores, rel=1e-5):
    """Index sets may differ only by elements whose (oracle) score is within
    rel of the boundary score of the oracle selection."""
    got, want = set(map(int, got_idx)), set(map(int, want_idx))
    if got == want:
        return
    boundary = min(scores[j] for j in want)
    tol = rel * max(1.0, abs(boundary))
    for j in got ^ want:
        assert abs(scores[j] - boundary) <= tol, (j, scores[j], boundary)


# ------------------------------------------------------------------ K9 ---
@pytest.mark.parametrize("V,d,dtype", [(257, 1024, torch.float32), (300, 2048, torch.bfloat16),
                                       (33, 9, torch.float32), (64, 130, torch.bfloat16)])
def test_quantize_int4_bitexact(H, O, V, d, dtype):
    w = _data.rng(1).standard_normal((V, d), dtype=np.float32)
    w[3] = 0.0  # zero row -> scale 1 (approx.hpp:59)
    w[5, :3] = [7.0, -7.0, 3.5]
    if dtype == torch.bfloat16:
        w = _data.bf16_round(w)
    z = H.ScoreMatrix(T(w, dtype))
    a = H.ApproxScorer.quantize(z)
    codes, scales = a.export_q4()
    c_ref, s_ref = O.quantize_int4(w)
    assert np.array_equal(scales.view(np.uint32), s_ref.view(np.uint32))
    assert np.array_equal(codes, c_ref)


# ------------------------------------------------------------------ K1 ---
@pytest.mark.parametrize("V,d,B", [(1000, 1024, 1), (513, 2048, 3), (77, 4096, 5), (100, 33, 2),
                                   (4099, 2048, 8), (300, 1024, 12), (200, 2048, 40),
                                   (100, 1024, 70), (50, 192, 3), (8192, 2048, 8)])
@pytest.mark.parametrize("phi", [0, 1])
def test_q4_scores_int8_bitexact(H, O, V, d, B, phi):
    w = _data.rng(V + d).standard_normal((V, d), dtype=np.float32)
    codes, scales = O.quantize_int4(w)
    a = H.ApproxScorer.quantized(codes, scales)
    x = _data.queries(B, d, 7, scale=1.0)
    got = N(a.scores(T(x), phi=phi, x_mode=H.X_INT8))
    for b in range(B):
        want = O.q4_scores_int8(codes, scales, x[b], phi)
        assert np.array_equal(got[b].view(np.uint32), want.view(np.uint32)), b


@pytest.mark.parametrize("V,d,B", [(1000, 1024, 5), (513, 2048, 3), (4099, 2048, 8)])
def test_q4_scores_int8_dp4a_path_bitexact(H, O, V, d, B, monkeypatch):
    """The CUDA-core dp4a kernel (HIRE_PROXY_KERNEL=dp4a) gives the same
    integers as the tensor-core kernel and the oracle."""
    monkeypatch.setenv("HIRE_PROXY_KERNEL", "dp4a")
    ctx = H.Context(0)
    w = _data.rng(V * 3 + d).standard_normal((V, d), dtype=np.float32)
    codes, scales = O.quantize_int4(w)
    a = H.ApproxScorer.quantized(codes, scales)
    x = _data.queries(B, d, 8, scale=1.0)
    got = N(a.scores(T(x), phi=0, x_mode=H.X_INT8, ctx=ctx))
    torch.cuda.synchronize()
    for b in range(B):
        want = O.q4_scores_int8(codes, scales, x[b], 0)
        assert np.array_equal(got[b].view(np.uint32), want.view(np.uint32)), b


@pytest.mark.parametrize("V,d", [(300, 1024), (129, 2048), (50, 70)])
def test_q4_scores_fpx_strict_bitexact_fast_close(H, O, V, d):
    w = _data.rng(d).standard_normal((V, d), dtype=np.float32)
    codes, scales = O.quantize_int4(w)
    a = H.ApproxScorer.quantized(codes, scales)
    x = _data.queries(2, d, 9)
    strict = N(a.scores(T(x), phi=1, strict=True))
    fast = N(a.scores(T(x), phi=1, strict=False))
    for b in range(2):
        want = O.q4_scores_fpx(codes, scales, x[b], 1)
        assert np.array_equal(strict[b].view(np.uint32), want.view(np.uint32))
        np.testing.assert_allclose(fast[b], want, rtol=1e-5, atol=1e-5 * np.abs(want).max())


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("r", [64, 7])
def test_lowrank_scores(H, O, dtype, r):
    V, d, B = 3000, 1024, 3
    g = _data.rng(r)
    z1 = g.standard_normal((r, d), dtype=np.float32)
    z2 = g.standard_normal((V, r), dtype=np.float32)
    if dtype == torch.bfloat16:
        z1, z2 = _data.bf16_round(z1), _data.bf16_round(z2)
    a = H.ApproxScorer.low_rank(T(z1, dtype), T(z2, dtype))
    x = _data.queries(B, d, 3)
    strict = N(a.scores(T(x), strict=True))
    fast = N(a.scores(T(x)))
    for b in range(B):
        want = O.lowrank_scores(z1, z2, x[b], 0)
        assert np.array_equal(strict[b].view(np.uint32), want.view(np.uint32))
        np.testing.assert_allclose(fast[b], want, rtol=1e-4, atol=1e-5 * np.abs(want).max())


# ------------------------------------------------------------------ K3 ---
@pytest.mark.parametrize("n,k", [(10, 3), (1000, 1000), (8192, 820), (32768, 256), (40000, 1024),
                                 (256000, 1024), (100000, 4000)])
def test_topk_select_matches_oracle_with_ties(H, O, n, k):
    g = _data.rng(n)
    v = g.integers(-50, 50, size=(2, n)).astype(np.float32)  # heavy ties
    v[1] = g.standard_normal(n).astype(np.float32)
    v[1, ::7] = 0.0
    v[1, 3::11] = -0.0  # -0 ties +0 (linalg.hpp:131)
    idx, val, cl = H.topk_select(T(v), k)
    for b in range(2):
        wi, wv, wcl = O.topk_select(v[b], k)
        assert np.array_equal(N(idx[b]).astype(np.uint32), wi)
        assert np.array_equal(N(val[b]), wv)
        assert cl == wcl


def test_topk_select_clamps(H, O):
    v = np.array([[3.0, 1.0, 2.0]], dtype=np.float32)
    idx, val, cl = H.topk_select(T(v), 5)
    assert cl and list(N(idx[0])) == [0, 2, 1]


# ------------------------------------------------------- hire_topk (K1-K5) ---
def _q4_instance(H, O, V, d, seed, dtype=torch.bfloat16):
    w = _data.lowrank_plus_noise(V, d, 32, seed)
    if dtype == torch.bfloat16:
        w = _data.bf16_round(w)
    codes, scales = O.quantize_int4(w)
    return w, H.ScoreMatrix(T(w, dtype)), H.ApproxScorer.quantized(codes, scales), codes, scales


@pytest.mark.parametrize("V,d,k,kp,B", [(4096, 1024, 32, 256, 3), (50000, 2048, 64, 1024, 2),
                                        (300, 64, 5, 40, 2)])
def test_hire_topk_int8_candidates_bitexact_strict_topk_bitexact(H, O, V, d, k, kp, B):
    w, z, a, codes, scales = _q4_instance(H, O, V, d, V)
    x = _data.queries(B, d, 11)
    cfg = H.HireConfig(k=k, k_prime=kp, phi="identity", x_mode=H.X_INT8, strict=True)
    r = H.hire_topk(T(x), z, a, cfg)
    for b in range(B):
        approx = O.q4_scores_int8(codes, scales, x[b], 0)
        o = O.hire_topk(w, x[b], approx, k, kp, 0)
        assert np.array_equal(N(r.cand[b]).astype(np.uint32), o["cand"])
        assert np.array_equal(N(r.top_idx[b]).astype(np.uint32), o["top_idx"])
        assert np.array_equal(N(r.top_val[b]).view(np.uint32), o["top_val"].view(np.uint32))


@pytest.mark.parametrize("V,d,k,kp", [(32768, 1024, 32, 256), (256000 // 8, 2048, 64, 1024)])
def test_hire_topk_fast_within_tolerance(H, O, V, d, k, kp):
    w, z, a, codes, scales = _q4_instance(H, O, V, d, 5)
    x = _data.queries(2, d, 12)
    r = H.hire_topk(T(x), z, a, H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8))
    for b in range(2):
        approx = O.q4_scores_int8(codes, scales, x[b], 0)
        o = O.hire_topk(w, x[b], approx, k, kp, 0)
        assert np.array_equal(N(r.cand[b]).astype(np.uint32), o["cand"])  # integer path
        exact = O.matvec(w, x[b])
        assert_sets_near_tie(N(r.top_idx[b]), o["top_idx"], exact)
        got_v = N(r.top_val[b])
        np.testing.assert_allclose(got_v, exact[N(r.top_idx[b])], rtol=1e-3, atol=1e-5)


def test_hire_topk_fpx_strict_equals_reference(H, O):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    V, d = 2000, 1024
    w, z, a, codes, scales = _q4_instance(H, O, V, d, 21, dtype=torch.float32)
    x = _data.queries(2, d, 13)
    rm, ra = O.RefMatrix(w), O.RefScorer("quantized", codes=codes, scales=scales)
    for phi in (0, 1, 2):
        r = H.hire_topk(T(x), z, a, H.HireConfig(k=16, k_prime=128, phi=phi, strict=True))
        for b in range(2):
            o = O.ref_hire_topk(rm, ra, x[b], 16, 128, phi)
            assert np.array_equal(N(r.cand[b]).astype(np.uint32), o["cand"])
            assert np.array_equal(N(r.top_idx[b]).astype(np.uint32), o["top_idx"])
            assert np.array_equal(N(r.top_val[b]).view(np.uint32), o["top_val"].view(np.uint32))


@pytest.mark.parametrize("nb,t,kp", [(1024, 1, 1024), (512, 2, 1024), (100, 3, 250), (7, 5, 30)])
def test_bucketed_literal_rule(H, O, nb, t, kp):
    V, d = 25600, 1024
    w, z, a, codes, scales = _q4_instance(H, O, V, d, 33)
    x = _data.queries(2, d, 14)
    cfg = H.HireConfig(k=min(64, kp), k_prime=kp, x_mode=H.X_INT8, select=H.SELECT_BUCKETED,
                       n_buckets=nb, bucket_t=t, strict=True)
    r = H.hire_topk(T(x), z, a, cfg)
    for b in range(2):
        approx = O.q4_scores_int8(codes, scales, x[b], 0)
        want, _ = O.bucketed_select(approx, nb, t, kp)
        assert np.array_equal(N(r.cand[b]).astype(np.uint32), want)
        o = O.hire_topk(w, x[b], approx, cfg.k, kp, 0, O.SEL_BUCKETED, nb, t)
        assert np.array_equal(N(r.top_idx[b]).astype(np.uint32), o["top_idx"])


def test_softmax_topk(H, O):
    V, d, k = 5000, 1024, 32
    w, z, a, codes, scales = _q4_instance(H, O, V, d, 44, dtype=torch.float32)
    x = _data.queries(3, d, 15, scale=0.5)
    idx, prob = H.softmax_topk(z, T(x), a, H.HireConfig(k=k, k_prime=256, strict=True))
    for b in range(3):
        approx = O.q4_scores_fpx(codes, scales, x[b], 0)
        o = O.hire_topk(w, x[b], approx, k, 256, 0)
        assert np.array_equal(N(idx[b]).astype(np.uint32), o["top_idx"])
        want = O.softmax_probs(o["top_val"])
        np.testing.assert_allclose(N(prob[b]), want, rtol=1e-6, atol=1e-7)
        assert abs(float(N(prob[b]).astype(np.float64).sum()) - 1.0) < 1e-5


def test_config_validation(H, O):
    w, z, a, codes, scales = _q4_instance(H, O, 64, 32, 1)
    x = T(_data.queries(1, 32, 1))
    with pytest.raises(H.HireInvalidArgument, match="k must be >= 1"):
        H.hire_topk(x, z, a, H.HireConfig(k=0, k_prime=4))
    with pytest.raises(H.HireInvalidArgument, match="must be <= k_prime"):
        H.hire_topk(x, z, a, H.HireConfig(k=5, k_prime=4))
    r = H.hire_topk(x, z, a, H.HireConfig(k=2, k_prime=100))  # clamps, hire.hpp:84
    assert r.clamped and r.cand.shape[1] == 64


# --------------------------------------------------------------- FFN (K6) ---
@pytest.mark.parametrize("g", [1, 2])
def test_ffn_group_sparse(H, O, g):
    m, d, k, kp, B = 2048, 1024, 102, 204, 3
    u, v = _data.ffn_family(m, d, 3, r=32)
    u, v = _data.bf16_round(u), _data.bf16_round(v)
    codes, scales = O.quantize_int4(u)
    f = H.GroupedFFN(H.ScoreMatrix(T(u, torch.bfloat16)), H.ScoreMatrix(T(v, torch.bfloat16)), g, "relu")
    a = H.ApproxScorer.quantized(codes, scales)
    x = _data.queries(B, d, 16, scale=1.0)
    out_s, sel_s = H.ffn_group_sparse(f, T(x), a, k, kp, x_mode=H.X_INT8, strict=True)
    out_f, sel_f = H.ffn_group_sparse(f, T(x), a, k, kp, x_mode=H.X_INT8, strict=False)
    for b in range(B):
        scores = O.q4_scores_int8(codes, scales, x[b], 1)
        ids, out = O.ffn_group_sparse(u, v, x[b], scores, k, kp, g, 1)
        assert np.array_equal(N(sel_s[b]).astype(np.uint32), ids)
        assert np.array_equal(N(out_s[b]).view(np.uint32), out.view(np.uint32))
        np.testing.assert_allclose(N(out_f[b]), out, rtol=1e-3, atol=1e-3 * np.abs(out).max())


def test_ffn_dense(H, O):
    m, d = 512, 1024
    u, v = _data.ffn_family(m, d, 4, r=16)
    f = H.GroupedFFN(H.ScoreMatrix(T(u)), H.ScoreMatrix(T(v)), 1, "relu")
    x = _data.queries(2, d, 17, scale=1.0)
    out = N(H.ffn_dense(f, T(x), strict=True))
    for b in range(2):
        want = O.ffn_dense(u, v, x[b], 1)
        assert np.array_equal(out[b].view(np.uint32), want.view(np.uint32))


# ------------------------------------------------------- DA-TOP-k (K7) ---
@pytest.mark.parametrize("s", [1, 2, 4, 8])
@pytest.mark.parametrize("merge", [0, 1])
def test_da_topk_emulated(H, O, s, merge):
    V, d, k, kp = 16000, 1024, 64, 512
    w, z, a, codes, scales = _q4_instance(H, O, V, d, 50 + s)
    x = _data.queries(2, d, 18)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8, strict=True)
    ti, tv, cl = H.da_topk_emulated(z, a, T(x), s, cfg, merge=merge)
    for b in range(2):
        scores = O.q4_scores_int8(codes, scales, x[b], 0)
        wi, wv, wcl, _ = O.da_topk(w, x[b], scores, s, k, kp, 0, merge=merge)
        assert np.array_equal(N(ti[b]).astype(np.uint32), wi)
        assert np.array_equal(N(tv[b]).view(np.uint32), wv.view(np.uint32))


def test_da_topk_uneven_quotas(H, O):
    V, d, k, kp, s = 9000, 1024, 410, 820, 8  # 8 does not divide 410 (cfg5)
    w, z, a, codes, scales = _q4_instance(H, O, V, d, 61)
    x = _data.queries(1, d, 19)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8, strict=True)
    with pytest.raises(H.HireInvalidArgument, match="must divide k"):
        H.da_topk_emulated(z, a, T(x), s, cfg)
    ti, tv, _ = H.da_topk_emulated(z, a, T(x), s, cfg, uneven=True)
    scores = O.q4_scores_int8(codes, scales, x[0], 0)
    wi, wv, _, _ = O.da_topk(w, x[0], scores, s, k, kp, 0, uneven=True)
    assert np.array_equal(N(ti[0]).astype(np.uint32), wi)


@pytest.mark.parametrize("s", [2, 4])
def test_da_group_sparse_emulated(H, O, s):
    m, d, k, kp = 2048, 1024, 128, 256
    u, v = _data.ffn_family(m, d, 8, r=32)
    codes, scales = O.quantize_int4(u)
    f = H.GroupedFFN(H.ScoreMatrix(T(u)), H.ScoreMatrix(T(v)), 1, "relu")
    a = H.ApproxScorer.quantized(codes, scales)
    x = _data.queries(2, d, 20, scale=1.0)
    out_s, sel_s = H.da_group_sparse_emulated(f, T(x), a, k, kp, s, x_mode=H.X_INT8, strict=True)
    out_f, _ = H.da_group_sparse_emulated(f, T(x), a, k, kp, s, x_mode=H.X_INT8)
    for b in range(2):
        scores = O.q4_scores_int8(codes, scales, x[b], 1)
        ids, out = O.da_group_sparse(u, v, x[b], scores, k, kp, s)
        assert np.array_equal(N(sel_s[b]).astype(np.uint32), ids)
        assert np.array_equal(N(out_s[b]).view(np.uint32), out.view(np.uint32))
        np.testing.assert_allclose(N(out_f[b]), out, rtol=1e-4, atol=1e-4 * np.abs(out).max())


@pytest.mark.parametrize("B", [1, 8, 13])
def test_ffn_fused_equals_unfused_and_oracle(H, O, B, monkeypatch):
    """The single-launch fused HiRE-FFN (cfg2 shape) is bit-identical to the
    unfused kernel chain, and matches the oracle (integer candidate step
    exact; final selection up to near-ties; outputs within 1e-3)."""
    if not H.lib().hire_experiments_built():
        pytest.skip("experiments-build kernel (-DHIRE_EXPERIMENTS=1)")
    m, d, k, kp = 8192, 2048, 410, 820
    u, v = _data.ffn_family(m, d, 40 + B, r=64)
    u, v = _data.bf16_round(u), _data.bf16_round(v)
    f = H.GroupedFFN(H.ScoreMatrix(T(u, torch.bfloat16)), H.ScoreMatrix(T(v, torch.bfloat16)), 1, "relu")
    a = H.ApproxScorer.quantize(f.u)
    codes, scales = a.export_q4()
    x = _data.queries(B, d, 41, scale=1.0)
    monkeypatch.setenv("HIRE_FFN_FUSED", "1")  # opt-in single-launch kernel (read at context creation)
    ctx_f = H.Context(0)
    out_f, sel_f = H.ffn_group_sparse(f, T(x), a, k, kp, x_mode=H.X_INT8, ctx=ctx_f)
    monkeypatch.setenv("HIRE_FFN_FUSED", "0")
    ctx = H.Context(0)
    out_u, sel_u = H.ffn_group_sparse(f, T(x), a, k, kp, x_mode=H.X_INT8, ctx=ctx)
    torch.cuda.synchronize()
    assert torch.equal(sel_f, sel_u)
    assert torch.equal(out_f.view(torch.int32), out_u.view(torch.int32))
    for b in range(B):
        s = O.q4_scores_int8(codes, scales, x[b], 1)
        ids, want = O.ffn_group_sparse(u, v, x[b], s, k, kp, 1, 1)
        acts = O.matvec(u, x[b], 1)
        assert_sets_near_tie(N(sel_f[b]), ids, acts)
        if set(N(sel_f[b]).tolist()) == set(ids.tolist()):
            np.testing.assert_allclose(N(out_f[b]), want, rtol=1e-3, atol=1e-3 * np.abs(want).max())


def test_recompute_bulk_copy_ring_equals_register_path(H, O, monkeypatch):
    if not H.lib().hire_experiments_built():
        pytest.skip("experiments-build kernel (-DHIRE_EXPERIMENTS=1)")
    # recompute_tma (opt-in) and recompute_fast share the arithmetic: identical values
    V, d, k, kp, B = 50000, 2048, 64, 1024, 9
    w, z, a, codes, scales = _q4_instance(H, O, V, d, 77)
    x = _data.queries(B, d, 78)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8)
    r0 = H.hire_topk(T(x), z, a, cfg)
    monkeypatch.setenv("HIRE_RECOMPUTE_TMA", "1")
    r1 = H.hire_topk(T(x), z, a, cfg)
    assert torch.equal(r0.top_idx, r1.top_idx)
    assert torch.equal(r0.top_val, r1.top_val)


@pytest.mark.parametrize("merge", [0, 1])
def test_da_topk_run_single_rank_equals_oracle(H, O, merge):
    # hire_da_topk_run with world = 1 (the bench's cfg4 at N = 1): one shard
    import paper_2402_09360_b200.parallel as P
    V, d, k, kp = 30000, 1024, 64, 512
    w, z, a, codes, scales = _q4_instance(H, O, V, d, 81)
    x = _data.queries(2, d, 82)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8, strict=True)
    ti, tv, cl = P.da_topk(z, a, V, T(x), cfg, None, merge=merge)
    for b in range(2):
        scores = O.q4_scores_int8(codes, scales, x[b], 0)
        wi, wv, wcl, _ = O.da_topk(w, x[b], scores, 1, k, kp, 0, merge=merge)
        assert np.array_equal(N(ti[b]).astype(np.uint32), wi)
        assert np.array_equal(N(tv[b]).view(np.uint32), wv.view(np.uint32))


def test_low_rank_quantized_scorer_equals_reference(H, O):
    # approx.hpp:342-347, 500-516 — against the compiled reference's own LRQ scorer
    if not O.ref_available():
        pytest.skip("compiled reference not built")
    g = np.random.default_rng(91)
    V, d, r = 5000, 256, 16
    z1 = g.standard_normal((r, d)).astype(np.float32)
    z2 = g.standard_normal((V, r)).astype(np.float32)
    x = _data.queries(3, d, 92)
    a = H.ApproxScorer.low_rank_quantized(T(z1), T(z2))
    got = N(a.scores(T(x), strict=True))
    ref = O.RefScorer("lrq", z1=z1, z2=z2)
    for b in range(3):
        assert np.array_equal(got[b].view(np.uint32), ref.scores(x[b], 0).view(np.uint32)), b


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_recompute_long_rows_equal_dense(H, O, dt):
    """d = 4096 (cfg4's rows; 16 lane chunks, one CTA/SM): gathered exact values equal the dense exact pass bit for bit
    (linalg.hpp:137-139 design rule) and a float64 recompute within 1e-5."""
    V, d, k, kp, B = 6000, 4096, 32, 700, 3
    w = _data.lowrank_plus_noise(V, d, 16, 41)
    z = H.ScoreMatrix(T(w).to(dt))
    codes, scales = O.quantize_int4(w)
    a = H.ApproxScorer.quantized(codes, scales)
    x = _data.queries(B, d, 42)
    r = H.hire_topk(T(x), z, a, H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8))
    dense = H.matvec(z, T(x))
    got = r.top_val.cpu()
    want = torch.gather(dense.cpu(), 1, r.top_idx.cpu().long())
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))
    wd = z.tensor.double().cpu() if hasattr(z, "tensor") else T(w).to(dt).double().cpu()
    ref = torch.from_numpy(x).double() @ wd.t()
    torch.testing.assert_close(got.double(), torch.gather(ref, 1, r.top_idx.cpu().long()), rtol=1e-5, atol=1e-5)
