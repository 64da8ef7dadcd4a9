"""The paper's batch-level FFN levers (SURVEY.md §8 f, rank 2) through the
C ABI: union_group_select (ffn.hpp:237-253), ffn_common_path
(ffn.hpp:223-234), overlap_ratio (metrics.hpp:68-88). GPU tests compare with
the oracle in strict mode (bit-exact); overlap_ratio is host arithmetic and
is checked against the reference's own rules on CPU."""
import numpy as np
import pytest
import torch

from tests import _data


def test_overlap_ratio_rules():
    import paper_2402_09360_b200 as H
    assert H.overlap_ratio([[1, 2, 3], [1, 2, 3]], 3) == pytest.approx(0.5)   # identical: 1/s
    assert H.overlap_ratio([[1, 2], [3, 4], [5, 6]], 2) == pytest.approx(1.0)  # disjoint: 1
    assert H.overlap_ratio([[0, 5], [5, 9]], 2) == pytest.approx(0.75)
    with pytest.raises(H.HireInvalidArgument, match="no sample sets"):
        H.overlap_ratio([], 2)
    with pytest.raises(H.HireInvalidArgument, match="k_groups must be >= 1"):
        H.overlap_ratio([[1]], 0)
    with pytest.raises(H.HireInvalidArgument, match="sample selected 1 groups, expected 2"):
        H.overlap_ratio([[1, 2], [3]], 2)


def _ffn(H, m, d, seed, g=1):
    u, v = _data.ffn_family(m, d, seed, r=32)
    f = H.GroupedFFN(H.ScoreMatrix(torch.from_numpy(u).cuda()), H.ScoreMatrix(torch.from_numpy(v).cuda()), g)
    return f, u, v


@pytest.mark.gpu
@pytest.mark.parametrize("g", [1, 4])
def test_union_group_select(H, O, g):
    m, d, k, kp, B = 4096, 512, 256, 512, 5
    f, u, v = _ffn(H, m, d, 3 + g, g)
    a = H.ApproxScorer.quantize(f.u)
    codes, scales = a.export_q4()
    x = np.random.default_rng(g).standard_normal((B, d)).astype(np.float32)
    got = H.union_group_select(f, torch.from_numpy(x).cuda(), a, k, kp, x_mode=H.X_INT8, strict=True)
    want, per = set(), []
    for b in range(B):
        ids, _ = O.ffn_group_sparse(u, v, x[b], O.q4_scores_int8(codes, scales, x[b], 1), k, kp, g, 1)
        want |= set(map(int, ids))
        per.append(ids)
    assert np.array_equal(got, np.array(sorted(want), dtype=np.uint32))
    r = H.overlap_ratio(per, k // g)
    assert r == pytest.approx(len(want) / (B * (k // g)))


@pytest.mark.gpu
@pytest.mark.parametrize("dense_m", [0, 512])
def test_ffn_common_path_strict(H, O, dense_m):
    m, d, k, kp, B = 2048, 512, 102, 204, 2
    f, u, v = _ffn(H, m, d, 11)
    a = H.ApproxScorer.quantize(f.u)
    codes, scales = a.export_q4()
    dense = None
    if dense_m:
        du, dv = _data.ffn_family(dense_m, d, 12, r=16)
        dense = H.GroupedFFN(H.ScoreMatrix(torch.from_numpy(du).cuda()), H.ScoreMatrix(torch.from_numpy(dv).cuda()))
    x = np.random.default_rng(13).standard_normal((B, d)).astype(np.float32)
    out = H.ffn_common_path(H.CommonPathFFN(dense, f), torch.from_numpy(x).cuda(), a, k, kp, x_mode=H.X_INT8,
                            strict=True)
    for b in range(B):
        _, sp = O.ffn_group_sparse(u, v, x[b], O.q4_scores_int8(codes, scales, x[b], 1), k, kp, 1, 1)
        want = (O.ffn_dense(du, dv, x[b], 1) if dense_m else np.zeros(d, np.float32)).astype(np.float32)
        want = (want + sp).astype(np.float32)  # ffn.hpp:232: out[i] += sparse.output[i]
        assert np.array_equal(out[b].cpu().numpy().view(np.uint32), want.view(np.uint32)), b
