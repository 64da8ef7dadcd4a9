"""K1 on the 5th-generation tensor cores (score_umma.cuh: TMA ring ->
int4-to-u8 in registers -> TMEM A operand -> tcgen05.mma kind::i8 -> TMEM
accumulators -> epilogue) against the oracle's integer scorer, bit for bit.
Reference op: approx.hpp:395-403 in BASELINE's int8-x integer mode."""
import numpy as np
import pytest
import torch

from tests import _data

pytestmark = pytest.mark.gpu


def T(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dtype)


def _check(O, got, codes, scales, x, phi):
    for b in range(x.shape[0]):
        want = O.q4_scores_int8(codes, scales, x[b], phi)
        assert np.array_equal(got[b].view(np.uint32), want.view(np.uint32)), b


@pytest.mark.parametrize("V,d,B", [(128, 256, 9), (300, 2048, 16), (1000, 1024, 17), (4099, 2048, 32),
                                   (777, 512, 33), (2000, 2048, 48), (640, 2048, 64), (513, 4096, 32),
                                   (37965, 1024, 24)])
@pytest.mark.parametrize("phi", [0, 1])
def test_umma_scores_bitexact(H, O, V, d, B, phi):
    w = _data.rng(V * 7 + d + B).standard_normal((V, d), dtype=np.float32)
    w[1] = 0.0
    codes, scales = O.quantize_int4(w)
    a = H.ApproxScorer.quantized(codes, scales)
    x = _data.queries(B, d, 11, scale=1.0)
    x[0, :5] = [100.0, -100.0, 0.0, 3.0, -3.0]  # saturating codes of x
    got = a.scores(T(x), phi=phi, x_mode=H.X_INT8).cpu().numpy()
    _check(O, got, codes, scales, x, phi)


def test_umma_device_quantized_and_sliced(H, O):
    """Device-built proxy (K9) and DA-style row slices: a slice at a 128-row
    boundary shares the parent's tensor-core layout, any other builds its own."""
    V, d, B = 3000, 2048, 20
    w = _data.bf16_round(_data.rng(5).standard_normal((V, d), dtype=np.float32))
    z = H.ScoreMatrix(T(w, torch.bfloat16))
    a = H.ApproxScorer.quantize(z)
    codes, scales = a.export_q4()
    x = _data.queries(B, d, 12, scale=1.0)
    _check(O, a.scores(T(x), x_mode=H.X_INT8).cpu().numpy(), codes, scales, x, 0)
    for first, count in [(1280, 1000), (1000, 1500), (0, 129)]:
        s = a.slice_cols(first, count)
        got = s.scores(T(x), x_mode=H.X_INT8).cpu().numpy()
        _check(O, got, codes[first:first + count], scales[first:first + count], x, 0)


def test_umma_full_vocab_cfg3_b32(H, O):
    """cfg3 shape (V=256000, d=2048) at B=32: every row block of the
    persistent grid (2000 blocks over 148 CTAs), bit-exact on sampled rows
    plus a checksum of all scores against the oracle's."""
    V, d, B = 256000, 2048, 32
    g = torch.Generator(device="cuda").manual_seed(3)
    W = (torch.randn(V, d, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    z = H.ScoreMatrix(W)
    a = H.ApproxScorer.quantize(z)
    codes, scales = a.export_q4()
    x = _data.queries(B, d, 13, scale=1.0)
    got = a.scores(T(x), x_mode=H.X_INT8).cpu().numpy()
    for b in (0, 17, 31):
        want = O.q4_scores_int8(codes, scales, x[b], 0)
        assert np.array_equal(got[b].view(np.uint32), want.view(np.uint32)), b


# ---- hire_topk on the tcgen05 proxy (9..64 queries): candidates through the selector ---
def _inst(H, O, V, d, seed, kind="lowrank"):
    if kind == "lowrank":
        w = _data.lowrank_plus_noise(V, d, 32, seed)
    elif kind == "int_ties":
        g = np.random.default_rng(seed)
        w = g.integers(-7, 8, size=(V, d)).astype(np.float32)
        w[:, 0] = 7.0
    else:  # equal rows: every score ties
        g = np.random.default_rng(seed)
        w = np.tile(g.standard_normal((1, d)).astype(np.float32), (V, 1))
    codes, scales = O.quantize_int4(w)
    return w, H.ScoreMatrix(T(w)), H.ApproxScorer.quantized(codes, scales), codes, scales


def _want(O, codes, scales, x, kp):
    idx, _, _ = O.topk_select(O.q4_scores_int8(codes, scales, x, 0), kp)
    return np.sort(idx.astype(np.uint32))


@pytest.mark.parametrize("V,d,kp,B", [(100000, 256, 1024, 9), (256000, 256, 1024, 32), (60000, 512, 4000, 17),
                                      (200000, 256, 2048, 64), (30001, 256, 512, 12)])
def test_umma_topk_candidates_bitexact(H, O, V, d, kp, B):
    w, z, a, codes, scales = _inst(H, O, V, d, V + B)
    x = _data.queries(B, d, V + 1)
    r = H.hire_topk(T(x), z, a, H.HireConfig(k=16, k_prime=kp, x_mode=H.X_INT8))
    for b in range(B):
        assert np.array_equal(r.cand[b].cpu().numpy().astype(np.uint32), _want(O, codes, scales, x[b], kp)), b


@pytest.mark.parametrize("kind", ["int_ties", "equal_rows"])
def test_umma_topk_ties_and_fallback(H, O, kind):
    V, d, kp, B = 40000, 256, 700, 12
    w, z, a, codes, scales = _inst(H, O, V, d, 4, kind)
    x = np.round(_data.queries(B, d, 5, scale=3.0)).astype(np.float32)
    x[2] = 0.0  # all-zero query: every score 0, ties broken by index
    r = H.hire_topk(T(x), z, a, H.HireConfig(k=4, k_prime=kp, x_mode=H.X_INT8))
    for b in range(B):
        assert np.array_equal(r.cand[b].cpu().numpy().astype(np.uint32), _want(O, codes, scales, x[b], kp)), b


def test_umma_topk_graph_replay(H, O):
    """zero-at-rest selector state under CUDA-graph replay, an all-zero
    query (exact fallback) inside a replay"""
    V, d, kp, B = 150000, 256, 1024, 24
    w, z, a, codes, scales = _inst(H, O, V, d, 8)
    cfg = H.HireConfig(k=64, k_prime=kp, x_mode=H.X_INT8)
    x = _data.queries(B, d, 9)
    g = np.random.default_rng(11)
    xd = T(x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        H.hire_topk(xd, z, a, cfg)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            r = H.hire_topk(xd, z, a, cfg)
    for it in range(4):
        xh = (g.standard_normal((B, d)) / np.sqrt(d)).astype(np.float32)
        if it == 2:
            xh[5] = 0.0
        xd.copy_(T(xh))
        graph.replay()
        torch.cuda.synchronize()
        for b in range(B):
            assert np.array_equal(r.cand[b].cpu().numpy().astype(np.uint32), _want(O, codes, scales, xh[b], kp)), (it, b)
