"""GPU: the batch-union gather recompute (exact.cuh K4U; the device side of
union_group_select's premise, ffn.hpp:237-253 — a row selected by several
inputs of a batch is fetched once) against the per-query gather and the
oracle. The union path sums per-512-byte-slice butterflies in slice order, so
its values agree with the per-query path to fp32 rounding, not bit for bit:
FFN outputs within 1e-5 relative (fp32 rows) / 1e-3 (bf16), selections equal
except at near-ties (|delta activation| <= 1e-5 relative), as BASELINE.json
allows for floating-point paths. The path is an experiments-build kernel
(measured slower than the per-query gather on B200, whose rows already leave
HBM once per batch — exact.cuh K4U): HIRE_UNION=1 switches it on there; the
product build skips these tests."""
import numpy as np
import pytest
import torch

from tests import _data

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _experiments_only(H):
    if not H.lib().hire_experiments_built():
        pytest.skip("batch-union gather: experiments build only (-DHIRE_EXPERIMENTS=1)")


def _ffn(H, m, d, seed, dtype=torch.float32, r=32):
    u, v = _data.ffn_family(m, d, seed, r=r)
    ut, vt = torch.from_numpy(u).cuda().to(dtype), torch.from_numpy(v).cuda().to(dtype)
    f = H.GroupedFFN(H.ScoreMatrix(ut), H.ScoreMatrix(vt), 1)
    return f, ut.float().cpu().numpy(), vt.float().cpu().numpy()


def _near_tie_equal(sel1, sel0, act_of, rel=1e-5):
    """selections equal, or differing only in units whose activations tie to rel"""
    bad = 0
    for b in range(sel1.shape[0]):
        s1, s0 = set(map(int, sel1[b])), set(map(int, sel0[b]))
        if s1 == s0:
            continue
        a = act_of(b)
        d1, d0 = sorted(s1 - s0), sorted(s0 - s1)
        assert len(d1) == len(d0)
        for p, q in zip(d1, d0):
            assert abs(a[p] - a[q]) <= rel * max(abs(a[p]), abs(a[q]), 1e-30), (b, p, q, a[p], a[q])
        bad += len(d1)
    return bad


@pytest.mark.parametrize("dtype,B", [(torch.float32, 16), (torch.bfloat16, 64), (torch.bfloat16, 17)])
def test_union_ffn_equals_per_query_path(H, O, monkeypatch, dtype, B):
    m, d, k, kp = 4096, 1024, 204, 408
    f, u, v = _ffn(H, m, d, 21, dtype)
    a = H.ApproxScorer.quantize(f.u)
    x = torch.from_numpy(np.random.default_rng(2).standard_normal((B, d)).astype(np.float32)).cuda()
    monkeypatch.setenv("HIRE_UNION", "1")
    o1, s1 = H.ffn_group_sparse(f, x, a, k, kp, x_mode=H.X_INT8)
    monkeypatch.setenv("HIRE_UNION", "0")
    o0, s0 = H.ffn_group_sparse(f, x, a, k, kp, x_mode=H.X_INT8)
    xa = x.cpu().numpy().astype(np.float64)
    flips = _near_tie_equal(s1.cpu().numpy(), s0.cpu().numpy(),
                            lambda b: np.maximum(u.astype(np.float64) @ xa[b], 0.0))
    assert flips <= 2
    tol = 1e-5 if dtype == torch.float32 else 1e-3
    scale = float(o0.abs().max())
    assert float((o1 - o0).abs().max()) <= tol * scale


def test_union_ffn_matches_oracle_fp32(H, O, monkeypatch):
    m, d, k, kp, B = 2048, 512, 102, 204, 24
    f, u, v = _ffn(H, m, d, 5)
    a = H.ApproxScorer.quantize(f.u)
    codes, scales = a.export_q4()
    x = np.random.default_rng(9).standard_normal((B, d)).astype(np.float32)
    monkeypatch.setenv("HIRE_UNION", "1")
    out, sel = H.ffn_group_sparse(f, torch.from_numpy(x).cuda(), a, k, kp, x_mode=H.X_INT8)
    out, sel = out.cpu().numpy(), sel.cpu().numpy()
    for b in range(B):
        ids, want = O.ffn_group_sparse(u, v, x[b], O.q4_scores_int8(codes, scales, x[b], 1), k, kp, 1, 1)
        if set(map(int, ids)) == set(map(int, sel[b])):
            np.testing.assert_allclose(out[b], want, rtol=1e-5, atol=1e-5 * float(np.abs(want).max()))
        else:  # a near-tie at the k-th activation
            act = np.maximum(u.astype(np.float64) @ x[b].astype(np.float64), 0.0)
            for p, q in zip(sorted(set(map(int, ids)) - set(map(int, sel[b]))),
                            sorted(set(map(int, sel[b])) - set(map(int, ids)))):
                assert abs(act[p] - act[q]) <= 1e-5 * max(act[p], act[q])


def test_union_graph_replay(H, monkeypatch):
    # the row masks are zero at rest, so a captured layer replays on new inputs
    monkeypatch.setenv("HIRE_UNION", "1")
    m, d, k, kp, B = 2048, 1024, 204, 408, 32
    f, u, v = _ffn(H, m, d, 33, torch.bfloat16)
    a = H.ApproxScorer.quantize(f.u)
    g = torch.Generator(device="cuda").manual_seed(1)
    xs = [torch.randn(B, d, device="cuda", generator=g) for _ in range(3)]
    buf = torch.empty(B, d, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        buf.copy_(xs[0])
        H.ffn_group_sparse(f, buf, a, k, kp, x_mode=H.X_INT8)
        s.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            out, sel = H.ffn_group_sparse(f, buf, a, k, kp, x_mode=H.X_INT8)
        got = []
        for x in xs:
            buf.copy_(x)
            gr.replay()
            s.synchronize()
            got.append((out.clone(), sel.clone()))
    monkeypatch.setenv("HIRE_UNION", "0")
    for x, (o1, s1) in zip(xs, got):
        o0, s0 = H.ffn_group_sparse(f, x, a, k, kp, x_mode=H.X_INT8)
        same = (s1 == s0).all(dim=1)
        assert int((~same).sum()) <= 1
        scale = float(o0.abs().max())
        assert float((o1[same] - o0[same]).abs().max()) <= 1e-3 * scale


def test_union_hire_topk_candidates_unchanged(H, monkeypatch):
    # the softmax path with heavily overlapping candidate lists: same
    # candidates (the proxy and selector are untouched), exact values equal to
    # fp32 rounding, top-k equal except at near-ties
    V, d, k, kp, B = 2048, 512, 32, 512, 16
    w = torch.from_numpy(_data.lowrank_plus_noise(V, d, 16, 3)).cuda()
    z = H.ScoreMatrix(w)
    a = H.ApproxScorer.quantize(z)
    x = torch.from_numpy(_data.queries(B, d, 4)).cuda()
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8)
    monkeypatch.setenv("HIRE_UNION", "1")
    r1 = H.hire_topk(x, z, a, cfg)
    monkeypatch.setenv("HIRE_UNION", "0")
    r0 = H.hire_topk(x, z, a, cfg)
    assert torch.equal(r1.cand, r0.cand)
    same = (r1.top_idx == r0.top_idx).all(dim=1)
    assert int((~same).sum()) <= 1
    torch.testing.assert_close(r1.top_val[same], r0.top_val[same], rtol=1e-5, atol=1e-6)
