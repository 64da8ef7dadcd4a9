"""The reference's weight files (HIRM io.hpp:94-107, HIRQ approx.hpp:551-586,
HIRL approx.hpp:588-608) loaded straight into device handles. CPU: the
parsers against bytes written by the compiled reference (HIRQ) and by the
reference's put_* layout, plus its IoError rules. GPU: loaded handles score
like the in-memory ones."""
import numpy as np
import pytest
import torch

from tests import _data


def test_parsers_and_errors(O, tmp_path):
    from paper_2402_09360_b200 import io
    g = np.random.default_rng(0)
    w = g.standard_normal((7, 5)).astype(np.float32)          # l = 7 columns of d = 5
    d, l, v = io.parse_matrix(io.format_matrix(w))
    assert (d, l) == (5, 7) and np.array_equal(v, w)
    z1 = g.standard_normal((3, 5)).astype(np.float32)
    z2 = g.standard_normal((7, 3)).astype(np.float32)
    a1, a2 = io.parse_low_rank(io.format_low_rank(z1, z2))
    assert np.array_equal(a1, z1) and np.array_equal(a2, z2)
    codes, scales = O.quantize_int4(w)
    if O.ref_available():  # HIRQ bytes written by the compiled reference itself
        import ctypes as C
        c8 = np.ascontiguousarray(codes, dtype=np.int8)
        buf = np.zeros(4096, dtype=np.uint8)
        n = O.ref().ref_write_quantized(c8.ctypes.data_as(C.c_void_p), scales.ctypes.data_as(C.c_void_p),
                                        7, 5, buf.ctypes.data_as(C.c_void_p), buf.size)
        rd, rl, payload, sc = io.parse_quantized(buf[:n].tobytes())
        assert (rd, rl) == (5, 7) and np.array_equal(sc, scales)
        assert np.array_equal(payload, O.pack_int4(codes.reshape(-1)))
    with pytest.raises(io.HireIoError, match="io: bad magic, expected HIRM"):
        io.parse_matrix(b"HIRQ" + bytes(8))
    with pytest.raises(io.HireIoError, match="io: truncated"):
        io.parse_matrix(io.format_matrix(w)[:-4])
    with pytest.raises(io.HireIoError, match="io: truncated HIRQ payload"):
        io.parse_quantized(b"HIRQ" + (5).to_bytes(4, "little") + (7).to_bytes(4, "little") + scales.tobytes() + b"\x00")
    with pytest.raises(io.HireIoError, match="io: cannot open for read"):
        io.read_matrix_file(str(tmp_path / "missing.hirm"))


@pytest.mark.gpu
def test_loaded_handles_score_like_in_memory(H, O, tmp_path):
    from paper_2402_09360_b200 import io
    V, d = 3001, 96  # odd total: a HIRQ byte straddles two columns
    w = _data.lowrank_plus_noise(V, d, 8, 5)
    codes, scales = O.quantize_int4(w)
    (tmp_path / "w.hirm").write_bytes(io.format_matrix(w))
    payload = O.pack_int4(codes.reshape(-1))
    (tmp_path / "p.hirq").write_bytes(b"HIRQ" + d.to_bytes(4, "little") + V.to_bytes(4, "little") +
                                      scales.astype("<f4").tobytes() + payload.tobytes())
    z = io.read_matrix_file(str(tmp_path / "w.hirm"))
    a = io.read_quantized_file(str(tmp_path / "p.hirq"))
    c2, s2 = a.export_q4()
    assert np.array_equal(c2, codes) and np.array_equal(s2, scales)
    x = _data.queries(2, d, 6)
    r = H.hire_topk(torch.from_numpy(x).cuda(), z, a, H.HireConfig(k=8, k_prime=64, strict=True))
    for b in range(2):
        o = O.hire_topk(w, x[b], O.q4_scores_fpx(codes, scales, x[b], 0), 8, 64, 0)
        assert np.array_equal(r.top_idx[b].cpu().numpy().astype(np.uint32), o["top_idx"])
    z1 = np.random.default_rng(7).standard_normal((8, d)).astype(np.float32)
    z2 = np.random.default_rng(8).standard_normal((V, 8)).astype(np.float32)
    (tmp_path / "f.hirl").write_bytes(io.format_low_rank(z1, z2))
    al = io.read_low_rank_file(str(tmp_path / "f.hirl"))
    s = al.scores(torch.from_numpy(x).cuda(), strict=True).cpu().numpy()
    for b in range(2):
        assert np.array_equal(s[b].view(np.uint32), O.lowrank_scores(z1, z2, x[b], 0).view(np.uint32))
