"""Generates tests/golden/*.npz from the reference itself.

Runs the UNMODIFIED reference headers (compiled behind a C shim into
oracle/_ref/libhire_ref.so by oracle/Makefile) on small seeded instances and
stores inputs + outputs. tests/test_oracle.py checks the C restatement
(oracle/liboracle.so) against these files, so the oracle stays pinned to the
reference even where /root/reference is absent (the GPU box).

  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def inst(V, d, seed):
    """Inputs from the reference's own generators (gen_instance kFlat and
    gen_vector, instance.hpp:16-21, 58-66), via the frozen Rng streams."""
    z = O.gen_gaussian(V * d, seed).reshape(V, d)  # column j = row j
    return z


def main():
    out = {}
    # rng streams (rng.hpp)
    for seed in (0, 42, 1234567, 20240201):
        u = np.empty(8, dtype=np.uint64)
        O.ref().ref_rng_u64(seed, 8, u.ctypes.data)
        f = np.empty(8, dtype=np.float64)
        O.ref().ref_rng_uniform(seed, 8, f.ctypes.data)
        g = np.empty(33, dtype=np.float32)
        O.ref().ref_gen_vector(33, seed, g.ctypes.data)
        out[f"rng_u64_{seed}"] = u
        out[f"rng_uniform_{seed}"] = f
        out[f"gen_vector_{seed}"] = g
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)

    cases = {}
    rng = np.random.default_rng(2024)
    for c in range(12):
        V = int(rng.integers(8, 300))
        d = int(rng.integers(1, 40))
        phi = int(rng.integers(0, 3))
        k = int(rng.integers(1, min(V, 20) + 1))
        kp = int(rng.integers(k, V + 3))
        w = inst(V, d, 100 + c)
        x = O.gen_gaussian(d, 500 + c)
        codes, scales = O.ref_quantize_int4(w)
        m = O.RefMatrix(w)
        a = O.RefScorer("quantized", codes=codes, scales=scales)
        r = O.ref_hire_topk(m, a, x, k, kp, phi)
        cases[f"q{c}"] = dict(w=w, x=x, phi=phi, k=k, kp=kp, codes=codes, scales=scales,
                              scores=a.scores(x, phi), cand=r["cand"], top_idx=r["top_idx"],
                              top_val=r["top_val"], clamped=r["clamped"])
        # low-rank scorer on the same instance
        rr = min(3, V, d)
        z1 = O.gen_gaussian(rr * d, 700 + c).reshape(rr, d)
        z2 = O.gen_gaussian(V * rr, 800 + c).reshape(V, rr)
        al = O.RefScorer("lowrank", z1=z1, z2=z2)
        rl = O.ref_hire_topk(m, al, x, k, kp, phi)
        cases[f"lr{c}"] = dict(w=w, x=x, phi=phi, k=k, kp=kp, z1=z1, z2=z2, scores=al.scores(x, phi),
                               cand=rl["cand"], top_idx=rl["top_idx"], top_val=rl["top_val"])
        # softmax (identity phi)
        si, sp = O.ref_softmax_topk(m, a, x, k, kp)
        cases[f"sm{c}"] = dict(w=w, x=x, k=k, kp=kp, codes=codes, scales=scales, idx=si, prob=sp)
    # FFN (g = 1, 2) and DA
    for c in range(6):
        g = 1 if c < 3 else 2
        m_units, d = 48, int(rng.integers(3, 20))
        u = inst(m_units, d, 900 + c)
        v = inst(m_units, d, 950 + c)
        x = O.gen_gaussian(d, 990 + c)
        codes, scales = O.ref_quantize_int4(u)
        f = O.RefFFN(u, v, g, 1)
        a = O.RefScorer("quantized", codes=codes, scales=scales)
        k, kp = 8 * g, 16 * g
        ids, outv = O.ref_ffn_group_sparse(f, a, x, k, kp)
        cases[f"ffn{c}"] = dict(u=u, v=v, x=x, g=g, k=k, kp=kp, codes=codes, scales=scales,
                                ids=ids, out=outv)
        s = 2
        dids, dout = O.ref_da_group_sparse(f, a, x, k, kp, s)
        cases[f"dgs{c}"] = dict(u=u, v=v, x=x, g=g, k=k, kp=kp, s=s, codes=codes, scales=scales,
                                ids=dids, out=dout)
    for c in range(6):
        V, d = 60, 7
        s = [1, 2, 3, 4, 2, 3][c]
        k, kp = 12, 24
        w = inst(V, d, 1200 + c)
        x = O.gen_gaussian(d, 1300 + c)
        codes, scales = O.ref_quantize_int4(w)
        m = O.RefMatrix(w)
        a = O.RefScorer("quantized", codes=codes, scales=scales)
        phi = c % 2
        ti, tv, cl, by = O.ref_da_topk(m, a, x, s, k, kp, phi)
        cases[f"da{c}"] = dict(w=w, x=x, s=s, k=k, kp=kp, phi=phi, codes=codes, scales=scales,
                               idx=ti, val=tv, bytes=by)
    flat = {}
    for name, dct in cases.items():
        for key, val in dct.items():
            flat[f"{name}__{key}"] = np.asarray(val)
    np.savez_compressed(os.path.join(HERE, "reference_cases.npz"), **flat)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
