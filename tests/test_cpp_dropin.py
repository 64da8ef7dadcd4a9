"""The C++ drop-in (include/hire_b200.hpp): reference-style call sites
compile against it (CPU), and on the GPU its results equal the oracle's."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp")
LIBDIR = os.path.join(ROOT, "paper_2402_09360_b200")


def _compile(out):
    from paper_2402_09360_b200 import build
    build.build()
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
           f"-L{LIBDIR}", "-l:libhire_cuda.so", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_header_compiles(tmp_path):
    _compile(str(tmp_path / "dropin"))


@pytest.mark.gpu
def test_dropin_matches_oracle(O, tmp_path):
    exe = str(tmp_path / "dropin")
    _compile(exe)
    g = np.random.default_rng(3)
    V, d, k, kp = 3000, 256, 16, 128
    w = g.standard_normal((V, d)).astype(np.float32)
    x = (g.standard_normal(d) / 16).astype(np.float32)
    f = tmp_path / "inst.bin"
    with open(f, "wb") as fh:
        fh.write(np.array([V, d, k, kp], dtype=np.uint32).tobytes())
        fh.write(w.tobytes())
        fh.write(x.tobytes())
    out = subprocess.run([exe, str(f)], capture_output=True, text=True, check=True).stdout
    lines = {l.split()[0]: l.split()[1:] for l in out.splitlines() if l.strip()}
    assert lines["trace"] == ["3", "0", "1", "2", "|", "2", "3", "0", "2"]  # test_hire.cpp:60-75
    assert "must be <= k_prime" in " ".join(lines["validate"])
    codes, scales = O.quantize_int4(w)
    s = O.q4_scores_fpx(codes, scales, x, 0)
    o = O.hire_topk(w, x, s, k, kp, 0)
    assert [int(c) for c in lines["cand"]] == o["cand"].tolist()
    top = [(int(p.split(":")[0]), np.float32(float(p.split(":")[1]))) for p in lines["top"]]
    assert [t[0] for t in top] == o["top_idx"].tolist()
    assert [t[1] for t in top] == o["top_val"].tolist()
    probs = [np.float32(float(p.split(":")[1])) for p in lines["prob"]]
    np.testing.assert_allclose(probs, O.softmax_probs(o["top_val"]), rtol=1e-6)
    di, dv, _, by = O.da_topk(w, x, s, 2, k - k % 2, kp - kp % 2, 0)
    assert [int(p.split(":")[0]) for p in lines["da"]] == di.tolist()
    assert int(lines["bytes"][0]) == by
    sr = O.q4_scores_fpx(codes, scales, x, 1)
    ids, fo = O.ffn_group_sparse(w, w, x, sr, k, kp, 1, 1)
    assert [int(i) for i in lines["ffn"]] == ids.tolist()
    assert np.array_equal(np.array([np.float32(float(v)) for v in lines["ffnout"]]), fo)
    dense = O.ffn_dense(w, w, x, 1)
    assert np.array_equal(np.array([np.float32(float(v)) for v in lines["dense"]]), dense)
    common = (dense + fo).astype(np.float32)  # ffn.hpp:232
    assert np.array_equal(np.array([np.float32(float(v)) for v in lines["common"]]), common)
    xn = (-x).astype(np.float32)
    ids_n, _ = O.ffn_group_sparse(w, w, xn, O.q4_scores_fpx(codes, scales, xn, 1), k, kp, 1, 1)
    union = sorted(set(ids.tolist()) | set(ids_n.tolist()))
    assert [int(i) for i in lines["union"]] == union
    assert float(lines["overlap"][0]) == pytest.approx(len(union) / (2 * k))
