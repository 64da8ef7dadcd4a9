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
