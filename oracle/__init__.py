"""Parity checkers for the HiRE CUDA path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the CPU baseline, never as the thing measured or shipped.

Two libraries live here:

* ``liboracle.so`` — ``hire_oracle.c``, a plain-C restatement of the
  reference algorithm (each function cites /root/reference file:line), plus
  the EXTENSIONS BASELINE.json asks for (int8-x scoring, the bucketed rule,
  uneven DA quotas, the global DA merge).
* ``_ref/libhire_ref.so`` — the unmodified reference headers compiled behind
  a C shim (``ref_shim.cpp``); "the reference itself, run here".

Both are wrapped with numpy-in / numpy-out helpers below. Arrays are
row-major ``W[l, d]`` (== the reference's column-major d x l ScoreMatrix).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhire_ref.so")

PHI = {"identity": 0, "relu": 1, "squared-relu": 2}
SEL_EXACT, SEL_BUCKETED = 0, 1
MERGE_PER_SHARD, MERGE_GLOBAL = 0, 1

_u64, _i32, _f32, _f64, _vp = C.c_uint64, C.c_int, C.c_float, C.c_double, C.c_void_p


def build(force: bool = False) -> None:
    """Compile liboracle.so (and _ref when /root/reference is mounted)."""
    if force or not os.path.exists(ORACLE_SO) or (
        os.path.isdir("/root/reference/proj/include") and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a):
    return a.ctypes.data_as(_vp) if a is not None else None


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float32)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(ORACLE_SO)
        L.orc_rng_u64.restype = _u64
        L.orc_rng_u64.argtypes = [_u64, _u64]
        L.orc_rng_uniform.restype = _f64
        L.orc_rng_uniform.argtypes = [_u64, _u64]
        L.orc_derive_seed.restype = _u64
        L.orc_derive_seed.argtypes = [_u64, _u64]
        L.orc_gen_gaussian_range.argtypes = [_u64, _u64, _u64, _vp]
        L.orc_column_score.restype = _f32
        L.orc_column_score.argtypes = [_vp, _vp, _u64, _i32]
        L.orc_matvec.argtypes = [_vp, _u64, _u64, _vp, _i32, _vp]
        L.orc_topk_select.restype = _u64
        L.orc_topk_select.argtypes = [_vp, _u64, _u64, _vp, _vp, _vp]
        L.orc_quantize_int4.argtypes = [_vp, _u64, _u64, _vp, _vp]
        L.orc_pack_int4.argtypes = [_vp, _u64, _vp]
        L.orc_unpack_int4.argtypes = [_vp, _u64, _vp]
        L.orc_round_bf16.restype = _f32
        L.orc_round_bf16.argtypes = [_f32]
        L.orc_round_bf16_array.argtypes = [_vp, _u64, _vp]
        L.orc_q4_scores_fpx.argtypes = [_vp, _vp, _u64, _u64, _vp, _i32, _vp]
        L.orc_quantize_x_int8.argtypes = [_vp, _u64, _vp, _vp]
        L.orc_q4_scores_int8.argtypes = [_vp, _vp, _u64, _u64, _vp, _i32, _vp]
        L.orc_lowrank_t.argtypes = [_vp, _u64, _u64, _vp, _vp]
        L.orc_lowrank_scores_from_t.argtypes = [_vp, _u64, _u64, _vp, _i32, _vp]
        L.orc_lowrank_scores.argtypes = [_vp, _vp, _u64, _u64, _u64, _vp, _i32, _vp]
        L.orc_bucketed_select.restype = _u64
        L.orc_bucketed_select.argtypes = [_vp, _u64, _u64, _u64, _u64, _vp, _vp]
        L.orc_hire_topk.restype = _i32
        L.orc_hire_topk.argtypes = [_vp, _u64, _u64, _vp, _vp, _u64, _u64, _i32, _i32,
                                    _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp]
        L.orc_softmax_topk_probs.argtypes = [_vp, _u64, _vp]
        L.orc_recall.restype = _f64
        L.orc_recall.argtypes = [_vp, _u64, _vp, _u64, _vp, _vp]
        L.orc_group_proxy.argtypes = [_vp, _u64, _u64, _vp]
        L.orc_select_groups.restype = _i32
        L.orc_select_groups.argtypes = [_vp, _u64, _u64, _u64, _i32, _vp, _vp, _u64, _u64, _vp, _vp]
        L.orc_ffn_apply_groups.argtypes = [_vp, _vp, _u64, _u64, _i32, _vp, _vp, _u64, _vp]
        L.orc_ffn_group_sparse.restype = _i32
        L.orc_ffn_group_sparse.argtypes = [_vp, _vp, _u64, _u64, _u64, _i32, _vp, _vp,
                                           _u64, _u64, _vp, _vp, _vp]
        L.orc_ffn_dense.argtypes = [_vp, _vp, _u64, _u64, _i32, _vp, _vp]
        L.orc_quota.restype = _u64
        L.orc_quota.argtypes = [_u64, _u64, _u64]
        L.orc_partition.argtypes = [_u64, _u64, _u64, _vp, _vp]
        L.orc_da_topk.restype = _i32
        L.orc_da_topk.argtypes = [_vp, _u64, _u64, _vp, _vp, _u64, _u64, _u64, _i32, _i32,
                                  _i32, _vp, _vp, _vp, _vp, _vp]
        L.orc_da_group_sparse.restype = _i32
        L.orc_da_group_sparse.argtypes = [_vp, _vp, _u64, _u64, _u64, _i32, _vp, _vp, _u64,
                                          _u64, _u64, _i32, _vp, _vp, _vp]
        L.orc_param_bytes.argtypes = [_u64, _u64, _u64, _u64, _vp]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The compiled reference (oracle/_ref). Raises if it was never built."""
    global _ref
    if _ref is None:
        build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_u64.argtypes = [_u64, _u64, _vp]
        L.ref_rng_uniform.argtypes = [_u64, _u64, _vp]
        L.ref_derive_seed.restype = _u64
        L.ref_derive_seed.argtypes = [_u64, _u64]
        L.ref_gen_vector.argtypes = [_u64, _u64, _vp]
        L.ref_gen_instance.restype = _i32
        L.ref_gen_instance.argtypes = [_u64, _u64, _u64, _i32, _vp]
        L.ref_matrix_create.restype = _vp
        L.ref_matrix_create.argtypes = [_vp, _u64, _u64]
        L.ref_matrix_destroy.argtypes = [_vp]
        L.ref_scorer_create.restype = _vp
        L.ref_scorer_create.argtypes = [_i32, _vp, _vp, _vp, _vp, _vp, _u64, _u64, _u64]
        L.ref_scorer_destroy.argtypes = [_vp]
        L.ref_quantize_int4.restype = _i32
        L.ref_quantize_int4.argtypes = [_vp, _u64, _u64, _vp, _vp]
        L.ref_write_quantized.restype = _u64
        L.ref_write_quantized.argtypes = [_vp, _vp, _u64, _u64, _vp, _u64]
        L.ref_round_bf16.restype = _f32
        L.ref_round_bf16.argtypes = [_f32]
        L.ref_scores.restype = _i32
        L.ref_scores.argtypes = [_vp, _vp, _u64, _i32, _vp]
        L.ref_matvec.restype = _i32
        L.ref_matvec.argtypes = [_vp, _vp, _u64, _i32, _vp]
        L.ref_topk_select.restype = _i32
        L.ref_topk_select.argtypes = [_vp, _u64, _u64, _vp, _vp, _vp, _vp]
        L.ref_hire_topk.restype = _i32
        L.ref_hire_topk.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _i32, _vp, _vp, _vp,
                                    _vp, _vp, _vp]
        L.ref_softmax_topk.restype = _i32
        L.ref_softmax_topk.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _vp, _vp, _vp]
        L.ref_hire_topk_batch.restype = _i32
        L.ref_hire_topk_batch.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _u64, _i32, _vp,
                                          _vp, _i32]
        L.ref_ffn_create.restype = _vp
        L.ref_ffn_create.argtypes = [_vp, _vp, _u64, _u64, _u64, _i32]
        L.ref_ffn_destroy.argtypes = [_vp]
        L.ref_ffn_group_sparse.restype = _i32
        L.ref_ffn_group_sparse.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _vp, _vp, _vp]
        L.ref_ffn_group_sparse_batch.restype = _i32
        L.ref_ffn_group_sparse_batch.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _u64, _vp,
                                                 _i32]
        L.ref_ffn_dense.restype = _i32
        L.ref_ffn_dense.argtypes = [_vp, _vp, _u64, _vp]
        L.ref_da_topk.restype = _i32
        L.ref_da_topk.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _u64, _i32, _vp, _vp, _vp,
                                  _vp, _vp]
        L.ref_da_group_sparse.restype = _i32
        L.ref_da_group_sparse.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _u64, _vp, _vp,
                                          _vp]
        L.ref_recall.restype = _f64
        L.ref_recall.argtypes = [_vp, _u64, _vp, _vp, _u64, _vp, _vp]
        L.ref_param_bytes.argtypes = [_u64, _u64, _u64, _u64, _vp]
        _ref = L
    return _ref


class RefError(RuntimeError):
    pass


def _ref_check(rc):
    if rc != 0:
        raise RefError(ref().ref_last_error().decode())


# ---------------------------------------------------------------- oracle ---
def gen_gaussian(n: int, seed: int, first: int = 0, threads: int = 0) -> np.ndarray:
    """gen_vector(n, seed) (instance.hpp:16-21), optionally a sub-range; big
    ranges are split across host threads (the stream is counter based)."""
    out = np.empty(n, dtype=np.float32)
    L = lib()
    if threads <= 1 or n < (1 << 22):
        L.orc_gen_gaussian_range(seed, first, n, _p(out))
        return out
    import concurrent.futures as cf
    step = ((n + threads - 1) // threads + 1) & ~1
    def job(s):
        cnt = min(step, n - s)
        view = out[s:s + cnt]
        L.orc_gen_gaussian_range(seed, first + s, cnt, view.ctypes.data_as(_vp))
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, range(0, n, step)))
    return out


def derive_seed(seed: int, stream: int) -> int:
    return lib().orc_derive_seed(seed, stream)


def rng_u64(seed: int, n: int) -> np.ndarray:
    L = lib()
    return np.array([L.orc_rng_u64(seed, i + 1) for i in range(n)], dtype=np.uint64)


def rng_uniform(seed: int, n: int) -> np.ndarray:
    L = lib()
    return np.array([L.orc_rng_uniform(seed, i + 1) for i in range(n)], dtype=np.float64)


def round_bf16(a) -> np.ndarray:
    a = _f(a)
    out = np.empty_like(a)
    lib().orc_round_bf16_array(_p(a), a.size, _p(out))
    return out


def quantize_int4(w):
    w = _f(w)
    rows, d = w.shape
    codes = np.empty((rows, d), dtype=np.int8)
    scales = np.empty(rows, dtype=np.float32)
    lib().orc_quantize_int4(_p(w), rows, d, _p(codes), _p(scales))
    return codes, scales


def pack_int4(codes) -> np.ndarray:
    c = np.ascontiguousarray(codes, dtype=np.int8).reshape(-1)
    out = np.empty((c.size + 1) // 2, dtype=np.uint8)
    lib().orc_pack_int4(_p(c), c.size, _p(out))
    return out


def unpack_int4(packed, n: int) -> np.ndarray:
    p = np.ascontiguousarray(packed, dtype=np.uint8)
    out = np.empty(n, dtype=np.int8)
    lib().orc_unpack_int4(_p(p), n, _p(out))
    return out


def column_score(w_row, x, phi=0) -> float:
    w_row, x = _f(w_row), _f(x)
    return lib().orc_column_score(_p(w_row), _p(x), x.size, phi)


def matvec(w, x, phi=0) -> np.ndarray:
    w, x = _f(w), _f(x)
    out = np.empty(w.shape[0], dtype=np.float32)
    lib().orc_matvec(_p(w), w.shape[0], w.shape[1], _p(x), phi, _p(out))
    return out


def topk_select(v, k):
    v = _f(v)
    kk = min(k, v.size)
    idx = np.empty(max(kk, 1), dtype=np.uint32)
    val = np.empty(max(kk, 1), dtype=np.float32)
    cl = C.c_int(0)
    n = lib().orc_topk_select(_p(v), v.size, k, _p(idx), _p(val), C.byref(cl))
    if n == (1 << 64) - 1:
        raise ValueError("topk_select: k must be >= 1")
    return idx[:n], val[:n], bool(cl.value)


def exact_topk(w, x, k, phi=0):
    return topk_select(matvec(w, x, phi), k)


def q4_scores_fpx(codes, scales, x, phi=0) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.int8)
    scales, x = _f(scales), _f(x)
    out = np.empty(codes.shape[0], dtype=np.float32)
    lib().orc_q4_scores_fpx(_p(codes), _p(scales), codes.shape[0], codes.shape[1], _p(x), phi, _p(out))
    return out


def quantize_x_int8(x):
    x = _f(x)
    xq = np.empty(x.size, dtype=np.int8)
    sx = C.c_float(0)
    lib().orc_quantize_x_int8(_p(x), x.size, _p(xq), C.byref(sx))
    return xq, np.float32(sx.value)


def q4_scores_int8(codes, scales, x, phi=0) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.int8)
    scales, x = _f(scales), _f(x)
    out = np.empty(codes.shape[0], dtype=np.float32)
    lib().orc_q4_scores_int8(_p(codes), _p(scales), codes.shape[0], codes.shape[1], _p(x), phi, _p(out))
    return out


def lowrank_scores(z1, z2, x, phi=0) -> np.ndarray:
    """z1: [r, d] (reference z1 columns), z2: [l, r]."""
    z1, z2, x = _f(z1), _f(z2), _f(x)
    r, d = z1.shape
    out = np.empty(z2.shape[0], dtype=np.float32)
    lib().orc_lowrank_scores(_p(z1), _p(z2), d, z2.shape[0], r, _p(x), phi, _p(out))
    return out


def lowrank_t(z1, x) -> np.ndarray:
    z1, x = _f(z1), _f(x)
    t = np.empty(z1.shape[0], dtype=np.float32)
    lib().orc_lowrank_t(_p(z1), z1.shape[1], z1.shape[0], _p(x), _p(t))
    return t


def bucketed_select(s, n_buckets, t, k_prime):
    s = _f(s)
    out = np.empty(max(k_prime, 1), dtype=np.uint32)
    cl = C.c_int(0)
    n = lib().orc_bucketed_select(_p(s), s.size, n_buckets, t, k_prime, _p(out), C.byref(cl))
    return out[:n], bool(cl.value)


def partition(n, parts, i):
    f, w = C.c_uint64(0), C.c_uint64(0)
    lib().orc_partition(n, parts, i, C.byref(f), C.byref(w))
    return f.value, w.value


def quota(k, s, i) -> int:
    return lib().orc_quota(k, s, i)


def hire_topk(w, x, approx, k, k_prime, phi=0, sel_mode=SEL_EXACT, n_buckets=1, bucket_t=1):
    """hire.hpp:50-86 given precomputed (phi'd) approximate scores.
    Returns dict(cand, top_idx, top_val, clamped)."""
    w, x, approx = _f(w), _f(x), _f(approx)
    rows, d = w.shape
    kp = min(k_prime, rows)
    cand = np.empty(max(kp, 1), dtype=np.uint32)
    ti = np.empty(max(k, 1), dtype=np.uint32)
    tv = np.empty(max(k, 1), dtype=np.float32)
    nc, nt, cl = C.c_uint64(0), C.c_uint64(0), C.c_int(0)
    rc = lib().orc_hire_topk(_p(w), rows, d, _p(x), _p(approx), k, k_prime, phi, sel_mode,
                             n_buckets, bucket_t, _p(cand), C.byref(nc), _p(ti), _p(tv),
                             C.byref(nt), C.byref(cl))
    if rc:
        raise ValueError("hire_topk: invalid config")
    return dict(cand=cand[:nc.value], top_idx=ti[:nt.value], top_val=tv[:nt.value],
                clamped=bool(cl.value))


def softmax_probs(top_val) -> np.ndarray:
    v = _f(top_val)
    out = np.empty_like(v)
    lib().orc_softmax_topk_probs(_p(v), v.size, _p(out))
    return out


def recall(cand_sorted, exact_idx):
    c = np.ascontiguousarray(cand_sorted, dtype=np.uint32)
    e = np.ascontiguousarray(exact_idx, dtype=np.uint32)
    h, t1 = C.c_uint64(0), C.c_int(0)
    r = lib().orc_recall(_p(c), c.size, _p(e), e.size, C.byref(h), C.byref(t1))
    return r, h.value, bool(t1.value)


def group_proxy(scores, g):
    s = _f(scores)
    out = np.empty(s.size // g, dtype=np.float32)
    lib().orc_group_proxy(_p(s), s.size, g, _p(out))
    return out


def ffn_group_sparse(u, v, x, scores, k, k_prime, g=1, phi=1):
    u, v, x, scores = _f(u), _f(v), _f(x), _f(scores)
    m, d = u.shape
    ids = np.empty(max(k // max(g, 1), 1), dtype=np.uint32)
    n = C.c_uint64(0)
    out = np.empty(d, dtype=np.float32)
    rc = lib().orc_ffn_group_sparse(_p(u), _p(v), m, d, g, phi, _p(x), _p(scores), k, k_prime,
                                    _p(ids), C.byref(n), _p(out))
    if rc:
        raise ValueError("ffn_group_sparse: invalid argument")
    return ids[:n.value], out


def ffn_apply_groups(u, v, x, ids, g=1, phi=1):
    u, v, x = _f(u), _f(v), _f(x)
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    out = np.empty(u.shape[1], dtype=np.float32)
    lib().orc_ffn_apply_groups(_p(u), _p(v), u.shape[1], g, phi, _p(x), _p(ids), ids.size, _p(out))
    return out


def ffn_dense(u, v, x, phi=1):
    u, v, x = _f(u), _f(v), _f(x)
    out = np.empty(u.shape[1], dtype=np.float32)
    lib().orc_ffn_dense(_p(u), _p(v), u.shape[0], u.shape[1], phi, _p(x), _p(out))
    return out


def da_topk(w, x, scores, s, k, k_prime, phi=0, merge=MERGE_PER_SHARD, uneven=False):
    w, x, scores = _f(w), _f(x), _f(scores)
    rows, d = w.shape
    cap = k_prime + k + 1
    ti = np.empty(cap, dtype=np.uint32)
    tv = np.empty(cap, dtype=np.float32)
    n, cl, by = C.c_uint64(0), C.c_int(0), C.c_uint64(0)
    rc = lib().orc_da_topk(_p(w), rows, d, _p(x), _p(scores), s, k, k_prime, phi, merge,
                           int(uneven), _p(ti), _p(tv), C.byref(n), C.byref(cl), C.byref(by))
    if rc:
        raise ValueError("da_topk: invalid argument")
    return ti[:n.value], tv[:n.value], bool(cl.value), by.value


def da_group_sparse(u, v, x, scores, k, k_prime, s, g=1, phi=1, uneven=False):
    u, v, x, scores = _f(u), _f(v), _f(x), _f(scores)
    m, d = u.shape
    ids = np.empty(k // g + s + 1, dtype=np.uint32)
    n = C.c_uint64(0)
    out = np.empty(d, dtype=np.float32)
    rc = lib().orc_da_group_sparse(_p(u), _p(v), m, d, g, phi, _p(x), _p(scores), k, k_prime, s,
                                   int(uneven), _p(ids), C.byref(n), _p(out))
    if rc:
        raise ValueError("da_group_sparse: invalid argument")
    return ids[:n.value], out


def param_bytes(d, l, r, k_prime):
    out = np.zeros(4, dtype=np.uint64)
    lib().orc_param_bytes(d, l, r, k_prime, _p(out))
    return out


# -------------------------------------------------------------- reference --
class RefMatrix:
    def __init__(self, w):
        w = _f(w)
        self.rows, self.d = w.shape
        self.h = ref().ref_matrix_create(_p(w), self.rows, self.d)
        if not self.h:
            raise RefError(ref().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_matrix_destroy(self.h)


class RefScorer:
    """kind: 'exact' (needs matrix), 'lowrank' (z1 [r,d], z2 [l,r]),
    'quantized' (codes [l,d], scales [l]), 'lrq' (z1, z2)."""

    def __init__(self, kind, matrix=None, z1=None, z2=None, codes=None, scales=None):
        k = {"exact": 0, "lowrank": 1, "quantized": 2, "lrq": 3}[kind]
        self._keep = []
        cols = d = r = 0
        if k == 0:
            cols, d = matrix.rows, matrix.d
            self._keep.append(matrix)
        elif k in (1, 3):
            z1, z2 = _f(z1), _f(z2)
            r, d = z1.shape
            cols = z2.shape[0]
            self._keep += [z1, z2]
        else:
            codes = np.ascontiguousarray(codes, dtype=np.int8)
            scales = _f(scales)
            cols, d = codes.shape
            self._keep += [codes, scales]
        self.cols, self.d = cols, d
        self.h = ref().ref_scorer_create(k, matrix.h if k == 0 else None, _p(z1) if k in (1, 3) else None,
                                         _p(z2) if k in (1, 3) else None,
                                         _p(codes) if k == 2 else None,
                                         _p(scales) if k == 2 else None, cols, d, r)
        if not self.h:
            raise RefError(ref().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_scorer_destroy(self.h)

    def scores(self, x, phi=0):
        x = _f(x)
        out = np.empty(self.cols, dtype=np.float32)
        _ref_check(ref().ref_scores(self.h, _p(x), x.size, phi, _p(out)))
        return out


class RefFFN:
    def __init__(self, u, v, g=1, phi=1):
        u, v = _f(u), _f(v)
        self.m, self.d = u.shape
        self.h = ref().ref_ffn_create(_p(u), _p(v), self.m, self.d, g, phi)
        if not self.h:
            raise RefError(ref().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_ffn_destroy(self.h)


def ref_quantize_int4(w):
    w = _f(w)
    rows, d = w.shape
    codes = np.empty((rows, d), dtype=np.int8)
    scales = np.empty(rows, dtype=np.float32)
    _ref_check(ref().ref_quantize_int4(_p(w), rows, d, _p(codes), _p(scales)))
    return codes, scales


def ref_hire_topk(m: RefMatrix, a: RefScorer, x, k, k_prime, phi=0):
    x = _f(x)
    kp = min(k_prime, m.rows)
    cand = np.empty(max(kp, 1), dtype=np.uint32)
    ti = np.empty(max(k, 1), dtype=np.uint32)
    tv = np.empty(max(k, 1), dtype=np.float32)
    nc, nt, cl = C.c_uint64(0), C.c_uint64(0), C.c_int(0)
    _ref_check(ref().ref_hire_topk(m.h, a.h, _p(x), x.size, k, k_prime, phi, _p(cand),
                                   C.byref(nc), _p(ti), _p(tv), C.byref(nt), C.byref(cl)))
    return dict(cand=cand[:nc.value], top_idx=ti[:nt.value], top_val=tv[:nt.value],
                clamped=bool(cl.value))


def ref_softmax_topk(m: RefMatrix, a: RefScorer, x, k, k_prime):
    x = _f(x)
    idx = np.empty(k, dtype=np.uint32)
    pr = np.empty(k, dtype=np.float32)
    n = C.c_uint64(0)
    _ref_check(ref().ref_softmax_topk(m.h, a.h, _p(x), x.size, k, k_prime, _p(idx), _p(pr), C.byref(n)))
    return idx[:n.value], pr[:n.value]


def ref_ffn_group_sparse(f: RefFFN, a: RefScorer, x, k, k_prime):
    x = _f(x)
    ids = np.empty(max(k, 1), dtype=np.uint32)
    n = C.c_uint64(0)
    out = np.empty(f.d, dtype=np.float32)
    _ref_check(ref().ref_ffn_group_sparse(f.h, a.h, _p(x), x.size, k, k_prime, _p(ids), C.byref(n), _p(out)))
    return ids[:n.value], out


def ref_da_topk(m: RefMatrix, a: RefScorer, x, s, k, k_prime, phi=0):
    x = _f(x)
    ti = np.empty(k + 1, dtype=np.uint32)
    tv = np.empty(k + 1, dtype=np.float32)
    n, cl, by = C.c_uint64(0), C.c_int(0), C.c_uint64(0)
    _ref_check(ref().ref_da_topk(m.h, a.h, _p(x), x.size, s, k, k_prime, phi, _p(ti), _p(tv),
                                 C.byref(n), C.byref(cl), C.byref(by)))
    return ti[:n.value], tv[:n.value], bool(cl.value), by.value


def ref_da_group_sparse(f: RefFFN, a: RefScorer, x, k, k_prime, s):
    x = _f(x)
    ids = np.empty(k + s + 1, dtype=np.uint32)
    n = C.c_uint64(0)
    out = np.empty(f.d, dtype=np.float32)
    _ref_check(ref().ref_da_group_sparse(f.h, a.h, _p(x), x.size, k, k_prime, s, _p(ids),
                                         C.byref(n), _p(out)))
    return ids[:n.value], out
