"""Seeded synthetic inputs with BASELINE.json's weight families (small
shapes for parity). Both the CUDA path and the oracle get the same bytes."""
import numpy as np


def rng(seed):
    return np.random.default_rng(seed)


def lowrank_plus_noise(V, d, r, seed, lr_scale=1.0, noise=0.1):
    """W = lr_scale * A B / sqrt(r) + noise * N(0,1): unit-variance rank-r
    component (cfg3/cfg4 family)."""
    g = rng(seed)
    A = g.standard_normal((V, r), dtype=np.float32)
    B = g.standard_normal((r, d), dtype=np.float32)
    W = (A @ B) * np.float32(lr_scale / np.sqrt(r)) + np.float32(noise) * g.standard_normal((V, d), dtype=np.float32)
    return W.astype(np.float32)


def cfg1_family(V, d, seed):
    """cfg1: W = A B / 8 + 0.1 N(0,1) with A [V,64], B [64,d]; returns W and
    the rank-64 truncated-SVD factors z1 [64, d] = (U_r S_r)^T... in the
    reference's convention Z1 = U_r Sigma_r (d x r), Z2 = V_r (l x r)."""
    g = rng(seed)
    r = min(64, V, d)
    A = g.standard_normal((V, r), dtype=np.float32)
    Bm = g.standard_normal((r, d), dtype=np.float32)
    W = (A @ Bm) / np.float32(8.0) + np.float32(0.1) * g.standard_normal((V, d), dtype=np.float32)
    W = W.astype(np.float32)
    # Z (d x l) = W^T; SVD of Z: Z = U S Vt -> Z1 = U_r S_r (d x r), Z2 = Vt_r^T (l x r)
    U, S, Vt = np.linalg.svd(W.T.astype(np.float64), full_matrices=False)
    z1 = (U[:, :r] * S[:r]).T.astype(np.float32)         # [r, d]
    z2 = Vt[:r].T.astype(np.float32)                      # [l, r]
    return W, np.ascontiguousarray(z1), np.ascontiguousarray(z2)


def ffn_family(m, d, seed, r=128):
    """cfg2: U, V ~ N(0, 1/d) + 3 x a rank-r component of the same entry scale."""
    g = rng(seed)
    def one():
        base = g.standard_normal((m, d), dtype=np.float32) / np.float32(np.sqrt(d))
        A = g.standard_normal((m, r), dtype=np.float32)
        B = g.standard_normal((r, d), dtype=np.float32)
        return (base + np.float32(3.0) * (A @ B) / np.float32(np.sqrt(r * d))).astype(np.float32)
    return one(), one()


def queries(B, d, seed, scale=None):
    g = rng(seed)
    s = np.float32(1.0 / np.sqrt(d)) if scale is None else np.float32(scale)
    return (g.standard_normal((B, d), dtype=np.float32) * s).astype(np.float32)


def bf16_round(a):
    """round-to-nearest-even to bf16, widened back to fp32 (approx.hpp:76-81)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)
