"""CPU: pins the oracle (oracle/hire_oracle.c) before it is trusted.

1. The reference's own known-answer tests, restated (values cited from
   /root/reference/proj/tests/*.cpp).
2. Golden vectors produced by the reference itself (tests/golden/, generated
   by tests/golden/make_golden.py from oracle/_ref).
3. When oracle/_ref is built here, randomized differential checks against
   the reference directly.
"""
import math
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


# ------------------------------------------------ reference KATs, restated --
def test_rng_frozen_streams(O):
    # test_rng.cpp:13-27
    assert [int(v) for v in O.rng_u64(0, 4)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                0x06C45D188009454F, 0xF88BB8A8724C81EC]
    assert [int(v) for v in O.rng_u64(42, 2)] == [0xBDD732262FEB6E95, 0x28EFE333B266F103]
    assert [int(v) for v in O.rng_u64(1234567, 2)] == [0x599ED017FB08FC85, 0x2C73F08458540FA5]
    # test_rng.cpp:29-35
    assert list(O.rng_uniform(42, 4)) == [0.7415648787718233, 0.1599103928769201,
                                          0.27860113025513866, 0.34419071652363753]


def test_gaussian_moments(O):
    g = O.gen_gaussian(200000, 3).astype(np.float64)  # test_rng.cpp:51-62
    assert abs(g.mean()) < 0.01 and abs((g * g).mean() - 1.0) < 0.02


def test_quantize_int4_formula(O):
    # test_approx.cpp:94-107: [1,-2,3] -> scale 3/7, codes [2,-5,7]
    codes, scales = O.quantize_int4(np.array([[1.0, -2.0, 3.0]], dtype=np.float32))
    assert scales[0] == np.float32(3.0) / np.float32(7.0)
    assert list(codes[0]) == [2, -5, 7]
    # :109-115 zero column -> scale 1, codes 0
    codes, scales = O.quantize_int4(np.zeros((1, 2), dtype=np.float32))
    assert scales[0] == 1.0 and list(codes[0]) == [0, 0]
    # :117-127 representable values round-trip
    codes, scales = O.quantize_int4(np.array([[7.0, -7.0]], dtype=np.float32))
    assert scales[0] == 1.0 and list(codes[0]) == [7, -7]


def test_int4_score_12_over_7(O):
    # test_approx.cpp:298-309
    codes, scales = O.quantize_int4(np.array([[1.0, -2.0, 3.0]], dtype=np.float32))
    s = O.q4_scores_fpx(codes, scales, np.ones(3, dtype=np.float32), 0)
    assert abs(float(s[0]) - 12.0 / 7.0) < 1e-6


def test_round_trip_bound(O):
    w = np.random.default_rng(0).standard_normal((40, 33)).astype(np.float32)
    codes, scales = O.quantize_int4(w)
    err = np.abs(w - codes.astype(np.float32) * scales[:, None])
    assert np.all(err <= scales[:, None] / 2 + 1e-7)  # SPEC round-trip invariant


def test_hirq_nibble_packing(O):
    # test_io.cpp:79-93: codes [2, -5] pack to 0xB2 (low nibble first)
    assert O.pack_int4(np.array([2, -5], dtype=np.int8))[0] == 0xB2
    p = O.pack_int4(np.array([7, -7, 1], dtype=np.int8))  # odd count pads
    assert list(O.unpack_int4(p, 3)) == [7, -7, 1]


def test_round_bf16(O):
    assert O.round_bf16(np.array([1.0, 0.0, 1.0 + 2 ** -10], dtype=np.float32)).tolist() == [1.0, 0.0, 1.0]


def test_topk_tie_rules(O):
    # test_linalg.cpp:118-133
    idx, _, _ = O.topk_select(np.array([0.5, 0.25, 0.25], dtype=np.float32), 2)
    assert list(idx) == [0, 1]
    idx, val, _ = O.topk_select(np.array([5, 7, 7], dtype=np.float32), 2)
    assert list(idx) == [1, 2] and val[0] == 7.0
    idx, val, _ = O.topk_select(np.array([-1, -2], dtype=np.float32), 2)
    assert list(val) == [-1.0, -2.0]
    with pytest.raises(ValueError):
        O.topk_select(np.array([1.0], dtype=np.float32), 0)
    _, _, cl = O.topk_select(np.array([1, 2, 3], dtype=np.float32), 10)
    assert cl


def test_topk_full_sort_oracle_with_ties(O):
    # test_linalg.cpp:156-164: ties among values in {0..4}
    v = (O.rng_u64(12, 64) % np.uint64(5)).astype(np.float32)
    order = sorted(range(64), key=lambda i: (-v[i], i))
    for k in range(1, 65, 7):
        assert list(O.topk_select(v, k)[0]) == order[:k]


def test_hire_hand_trace(O):
    # test_hire.cpp:60-75: Z columns {(1,0),(0,1),(1,1),(-1,-1)}, x=(2,1),
    # approx [2.1,0.9,2.9,0], k=2, k'=3, ReLU -> S'={0,1,2}, {(2,3),(0,2)}
    w = np.array([[1, 0], [0, 1], [1, 1], [-1, -1]], dtype=np.float32)
    x = np.array([2, 1], dtype=np.float32)
    approx = np.array([2.1, 0.9, 2.9, 0.0], dtype=np.float32)
    r = O.hire_topk(w, x, np.maximum(approx, 0), 2, 3, 1)
    assert list(r["cand"]) == [0, 1, 2]
    assert list(r["top_idx"]) == [2, 0] and list(r["top_val"]) == [3.0, 2.0]
    # :79-94 missed argmax counterexample
    r = O.hire_topk(w, x, np.array([2.0, 1.5, 0.1, 0.2], dtype=np.float32), 1, 2, 1)
    assert list(r["top_idx"]) == [0]
    exact, _, _ = O.exact_topk(w, x, 1, 1)
    rec, hits, top1 = O.recall(r["cand"], exact)
    assert rec < 1.0 and not top1


def test_hire_config_validation(O):
    w = np.ones((8, 4), dtype=np.float32)
    x = np.ones(4, dtype=np.float32)
    with pytest.raises(ValueError):
        O.hire_topk(w, x, np.ones(8, np.float32), 0, 4)
    with pytest.raises(ValueError):
        O.hire_topk(w, x, np.ones(8, np.float32), 5, 4)
    r = O.hire_topk(w, x, np.ones(8, np.float32), 2, 100)  # clamp, hire.hpp:84
    assert r["clamped"] and r["cand"].size == 8


def test_softmax_closed_form(O):
    # test_hire.cpp:200-212: logits [ln2, 0, 0], k=2 -> {(0,2/3),(1,1/3)}
    w = np.array([[math.log(2.0)], [0.0], [0.0]], dtype=np.float32)
    x = np.ones(1, dtype=np.float32)
    r = O.hire_topk(w, x, O.matvec(w, x), 2, 2)
    assert list(r["top_idx"]) == [0, 1]
    p = O.softmax_probs(r["top_val"])
    assert abs(p[0] - 2 / 3) < 1e-6 and abs(p[1] - 1 / 3) < 1e-6


def test_ffn_hand_traces(O):
    # test_ffn.cpp:120-131 group proxy [1, 2]; :151-164 group-sparse trace
    u = np.array([[0.5, 0], [0, 0], [-1, -1], [1, 0]], dtype=np.float32)
    v = np.arange(8, dtype=np.float32).reshape(4, 2) + 1
    x = np.array([2, 1], dtype=np.float32)
    acts = O.matvec(u, x, 1)
    assert list(acts) == [1.0, 0.0, 0.0, 2.0]
    assert list(O.group_proxy(acts, 2)) == [1.0, 2.0]
    ids, out = O.ffn_group_sparse(u, v, x, acts, 2, 4, g=2, phi=1)
    assert list(ids) == [1]
    assert list(out) == [2.0 * v[3, 0], 2.0 * v[3, 1]]


def test_da_hand_traces(O):
    # test_distributed.cpp:69-102
    z = np.array([9, 1, 3, 7, 8, 2, 6, 4], dtype=np.float32)[:, None]
    x = np.ones(1, dtype=np.float32)
    ti, tv, _, _ = O.da_topk(z, x, O.matvec(z, x), 2, 2, 4)
    assert list(ti) == [0, 4] and list(tv) == [9.0, 8.0]
    z = np.array([9, 8, 1, 1, 2, 2, 2, 2], dtype=np.float32)[:, None]
    ti, tv, _, _ = O.da_topk(z, x, O.matvec(z, x), 2, 2, 4)
    assert list(ti) == [0, 4] and list(tv) == [9.0, 2.0]
    # the global-merge extension recovers the true top-2 here
    ti, tv, _, _ = O.da_topk(z, x, O.matvec(z, x), 2, 2, 4, merge=O.MERGE_GLOBAL)
    assert list(ti) == [0, 1]


def test_da_divisibility_and_uneven(O):
    z = np.arange(60, dtype=np.float32)[:, None]
    x = np.ones(1, dtype=np.float32)
    s = O.matvec(z, x)
    with pytest.raises(ValueError):
        O.da_topk(z, x, s, 3, 4, 8)  # 3 does not divide 4 (test_distributed.cpp:196-205)
    ti, _, _, _ = O.da_topk(z, x, s, 3, 4, 8, uneven=True)
    # quotas 2,1,1 over shards [0,20),[20,40),[40,60): 19,18 | 39 | 59
    assert sorted(ti.tolist()) == [18, 19, 39, 59]
    assert [O.quota(410, 8, i) for i in range(8)] == [52, 52, 51, 51, 51, 51, 51, 51]


def test_shard_width_rule(O):
    # test_distributed.cpp:38-48: l=10, s=3 -> widths 4,3,3 offsets 0,4,7
    assert [O.partition(10, 3, i) for i in range(3)] == [(0, 4), (4, 3), (7, 3)]


def test_recall_and_cost_model(O):
    # test_metrics.cpp:29-35 / :73-80
    rec, hits, top1 = O.recall(np.array([1, 2, 3, 4]), np.array([2, 5]))
    assert rec == 0.5 and hits == 1 and top1
    assert list(O.param_bytes(100, 1000, 10, 50)[:3]) == [200000, 32000, 60000]


def test_bucketed_rule_properties(O):
    g = np.random.default_rng(5)
    s = g.standard_normal(1000).astype(np.float32)
    # t >= bucket width -> every element survives -> exact top-k'
    got, cl = O.bucketed_select(s, 10, 100, 50)
    want, _, _ = O.topk_select(s, 50)
    assert list(got) == sorted(want.tolist()) and not cl
    # literal 1-per-bucket rule picks each bucket's argmax
    got, _ = O.bucketed_select(s, 50, 1, 50)
    assert list(got) == [20 * b + int(np.argmax(s[20 * b:20 * b + 20])) for b in range(50)]


def test_int8_mode_exact_when_representable(O):
    """Integer mode == the reference fp-x scorer whenever both are exact:
    integer weights with max |w| = 7 (scale 1) and integer x with max |x| =
    127 (sx = 1); every partial sum is an integer < 2^24."""
    g = np.random.default_rng(9)
    w = g.integers(-7, 8, size=(50, 64)).astype(np.float32)
    w[:, 0] = 7.0
    x = g.integers(-127, 128, size=64).astype(np.float32)
    x[0] = 127.0
    codes, scales = O.quantize_int4(w)
    assert np.all(scales == 1.0)
    for phi in (0, 1, 2):
        a = O.q4_scores_int8(codes, scales, x, phi)
        b = O.q4_scores_fpx(codes, scales, x, phi)
        assert np.array_equal(a, b)


# --------------------------------------------------- reference golden files --
def _cases():
    z = np.load(os.path.join(GOLD, "reference_cases.npz"))
    cases = {}
    for key in z.files:
        name, field = key.split("__")
        cases.setdefault(name, {})[field] = z[key]
    return cases


def test_golden_rng(O):
    z = np.load(os.path.join(GOLD, "rng.npz"))
    for seed in (0, 42, 1234567, 20240201):
        assert np.array_equal(O.rng_u64(seed, 8), z[f"rng_u64_{seed}"])
        assert np.array_equal(O.rng_uniform(seed, 8), z[f"rng_uniform_{seed}"])
        assert np.array_equal(O.gen_gaussian(33, seed), z[f"gen_vector_{seed}"])


def test_golden_reference_cases(O):
    cases = _cases()
    n = 0
    for name, c in cases.items():
        if name.startswith("q"):
            codes, scales = O.quantize_int4(c["w"])
            assert np.array_equal(codes, c["codes"]) and np.array_equal(scales, c["scales"]), name
            s = O.q4_scores_fpx(codes, scales, c["x"], int(c["phi"]))
            assert np.array_equal(s, c["scores"]), name
            r = O.hire_topk(c["w"], c["x"], s, int(c["k"]), int(c["kp"]), int(c["phi"]))
        elif name.startswith("lr"):
            s = O.lowrank_scores(c["z1"], c["z2"], c["x"], int(c["phi"]))
            assert np.array_equal(s, c["scores"]), name
            r = O.hire_topk(c["w"], c["x"], s, int(c["k"]), int(c["kp"]), int(c["phi"]))
        elif name.startswith("sm"):
            s = O.q4_scores_fpx(c["codes"], c["scales"], c["x"], 0)
            r = O.hire_topk(c["w"], c["x"], s, int(c["k"]), int(c["kp"]), 0)
            assert np.array_equal(r["top_idx"], c["idx"]), name
            assert np.array_equal(O.softmax_probs(r["top_val"]), c["prob"]), name
            n += 1
            continue
        elif name.startswith("ffn"):
            s = O.q4_scores_fpx(c["codes"], c["scales"], c["x"], 1)
            ids, out = O.ffn_group_sparse(c["u"], c["v"], c["x"], s, int(c["k"]), int(c["kp"]),
                                          int(c["g"]), 1)
            assert np.array_equal(ids, c["ids"]) and np.array_equal(out, c["out"]), name
            n += 1
            continue
        elif name.startswith("dgs"):
            s = O.q4_scores_fpx(c["codes"], c["scales"], c["x"], 1)
            ids, out = O.da_group_sparse(c["u"], c["v"], c["x"], s, int(c["k"]), int(c["kp"]),
                                         int(c["s"]), int(c["g"]), 1)
            assert np.array_equal(ids, c["ids"]) and np.array_equal(out, c["out"]), name
            n += 1
            continue
        elif name.startswith("da"):
            s = O.q4_scores_fpx(c["codes"], c["scales"], c["x"], int(c["phi"]))
            ti, tv, _, by = O.da_topk(c["w"], c["x"], s, int(c["s"]), int(c["k"]), int(c["kp"]),
                                      int(c["phi"]))
            assert np.array_equal(ti, c["idx"]) and np.array_equal(tv, c["val"]), name
            assert by == int(c["bytes"]), name
            n += 1
            continue
        else:
            continue
        assert np.array_equal(r["cand"], c["cand"]), name
        assert np.array_equal(r["top_idx"], c["top_idx"]), name
        assert np.array_equal(r["top_val"], c["top_val"]), name
        n += 1
    assert n == len(cases)


# ------------------------------------------- differential vs the reference --
@pytest.fixture(scope="module")
def R(O):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    return O


def test_differential_hire_topk(R):
    O = R
    g = np.random.default_rng(77)
    for trial in range(60):
        V, d = int(g.integers(2, 200)), int(g.integers(1, 50))
        w = g.standard_normal((V, d)).astype(np.float32)
        x = g.standard_normal(d).astype(np.float32)
        phi = int(g.integers(0, 3))
        k = int(g.integers(1, V + 1))
        kp = int(g.integers(k, V + 5))
        codes, scales = O.quantize_int4(w)
        m = O.RefMatrix(w)
        a = O.RefScorer("quantized", codes=codes, scales=scales)
        s = O.q4_scores_fpx(codes, scales, x, phi)
        assert np.array_equal(s, a.scores(x, phi))
        o, r = O.hire_topk(w, x, s, k, kp, phi), O.ref_hire_topk(m, a, x, k, kp, phi)
        for key in ("cand", "top_idx", "top_val", "clamped"):
            assert np.array_equal(o[key], r[key]), (trial, key)


def test_differential_ffn_and_da(R):
    O = R
    g = np.random.default_rng(78)
    for trial in range(20):
        gs = int(g.integers(1, 4))
        m, d = 12 * gs * 2, int(g.integers(2, 12))
        u = g.standard_normal((m, d)).astype(np.float32)
        v = g.standard_normal((m, d)).astype(np.float32)
        x = g.standard_normal(d).astype(np.float32)
        codes, scales = O.quantize_int4(u)
        f = O.RefFFN(u, v, gs, 1)
        a = O.RefScorer("quantized", codes=codes, scales=scales)
        s = O.q4_scores_fpx(codes, scales, x, 1)
        k, kp = 4 * gs, 8 * gs
        ids, out = O.ffn_group_sparse(u, v, x, s, k, kp, gs, 1)
        rids, rout = O.ref_ffn_group_sparse(f, a, x, k, kp)
        assert np.array_equal(ids, rids) and np.array_equal(out, rout)
        dids, dout = O.da_group_sparse(u, v, x, s, k, kp, 2, gs, 1)
        rdids, rdout = O.ref_da_group_sparse(f, a, x, k, kp, 2)
        assert np.array_equal(dids, rdids) and np.array_equal(dout, rdout)
        V = 40
        w = g.standard_normal((V, d)).astype(np.float32)
        wc, ws = O.quantize_int4(w)
        m_ = O.RefMatrix(w)
        aw = O.RefScorer("quantized", codes=wc, scales=ws)
        for sh in (1, 2, 4):
            sw = O.q4_scores_fpx(wc, ws, x, 0)
            ti, tv, cl, by = O.da_topk(w, x, sw, sh, 8, 16, 0)
            rti, rtv, rcl, rby = O.ref_da_topk(m_, aw, x, sh, 8, 16, 0)
            assert np.array_equal(ti, rti) and np.array_equal(tv, rtv) and by == rby


def test_differential_lowrank_and_quantize(R):
    O = R
    g = np.random.default_rng(79)
    for trial in range(20):
        V, d, r = int(g.integers(2, 300)), int(g.integers(1, 64)), int(g.integers(1, 9))
        w = g.standard_normal((V, d)).astype(np.float32)
        c1, s1 = O.quantize_int4(w)
        c2, s2 = O.ref_quantize_int4(w)
        assert np.array_equal(c1, c2) and np.array_equal(s1, s2)
        z1 = g.standard_normal((r, d)).astype(np.float32)
        z2 = g.standard_normal((V, r)).astype(np.float32)
        x = g.standard_normal(d).astype(np.float32)
        a = O.RefScorer("lowrank", z1=z1, z2=z2)
        for phi in (0, 1):
            assert np.array_equal(O.lowrank_scores(z1, z2, x, phi), a.scores(x, phi))
