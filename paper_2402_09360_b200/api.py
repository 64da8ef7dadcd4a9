"""Python mirror of the reference's `hire::` operator API for the hot path.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/hire/*.hpp so parity tests read like the
reference's own tests; every call goes through the C ABI of
libhire_cuda.so (include/hire_cuda.h). torch is only the device-memory and
stream plumbing. Batched: x is [B, d]; each query is an independent call of
the reference function.

Reference symbols mirrored (file:line under /root/reference/proj/include/hire):
  ScoreMatrix linalg.hpp:44 · topk_select :157 · matvec :148 · exact_topk :184
  ApproxScorer approx.hpp:327 (quantized :336, low_rank :332, slice_cols :415)
  quantize_int4 approx.hpp:49 · HireConfig hire.hpp:16 · hire_topk hire.hpp:50
  softmax_topk hire.hpp:123 · GroupedFFN ffn.hpp:19 · ffn_group_sparse :211
  ffn_dense :65 · shard distributed.hpp:41 · da_topk :73 · da_group_sparse :145
  recall metrics.hpp:23
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib as L
from ._lib import check, lib

_PHI = {"identity": 0, "relu": 1, "squared-relu": 2}


def _phi(p) -> int:
    return _PHI[p] if isinstance(p, str) else int(p)


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else None


class Context:
    """A hire_ctx bound to one CUDA stream (default: torch's current stream)."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        self.device = device
        s = stream if stream is not None else torch.cuda.current_stream(device)
        self.stream = s
        h = C.c_void_p()
        check(lib().hire_ctx_create(device, C.c_void_p(s.cuda_stream), 0, C.byref(h)))
        self.h = h

    def launches(self) -> int:
        return lib().hire_ctx_launch_count(self.h)

    def synchronize(self):
        check(lib().hire_ctx_synchronize(self.h))

    def select_fallbacks(self) -> int:
        """Queries whose exact top-k' selection took the slow whole-row path so
        far (hire_ctx_select_fallbacks): a time cliff, never a wrong result."""
        n = C.c_longlong()
        check(lib().hire_ctx_select_fallbacks(self.h, C.byref(n)))
        return int(n.value)

    def set_profiling(self, on: bool):
        check(lib().hire_ctx_set_profiling(self.h, int(on)))

    KT_NAMES = ["pivot", "window", "window_select", "emit", "final", "recompute", "proxy", "gather",
                "prep_x", "lr_t", "lr_score", "down"]

    def ktrace(self, op: int):
        """Debug kernel timeline (hire_debug_ktrace): op 1 enable+reset, 0 disable,
        2 -> {kernel: (start_us, end_us)} relative to the earliest start."""
        if op != 2:
            check(lib().hire_debug_ktrace(self.h, op, None, 0))
            return None
        buf = (C.c_ulonglong * 96)()
        check(lib().hire_debug_ktrace(self.h, 2, buf, 96))
        spans = {}
        for i, name in enumerate(self.KT_NAMES):
            a, b = buf[2 * i], buf[2 * i + 1]
            if b:
                spans[name] = (a, b)
        t0 = min(a for a, _ in spans.values()) if spans else 0
        if buf[39]:
            spans["emit_last_cta"] = (buf[39], buf[42])
            spans["emit_phases"] = (buf[40], buf[41])
            spans["emit_max_start_max_publish"] = (buf[43], buf[44])
        if buf[45]:
            spans["ws_counts"] = (buf[45], buf[46])
            spans["ws_bin"] = (buf[46], buf[47])
            if buf[48]:
                spans["ws_gather"] = (buf[47], buf[48])
                spans["ws_select"] = (buf[48], buf[49])
        if buf[52] or buf[55]:
            # fused proxy/filter kernel (fsel.cuh): sample arrivals, bracket
            # published, first/last CTA done streaming, last CTA done filtering
            if buf[52]:
                spans["fsel_sampled_bracket"] = (buf[52], buf[53] or buf[52])
            spans["proxy_cta_end_first_last"] = (buf[54], buf[55])
            if buf[56]:
                spans["fsel_filter_end"] = (buf[55], buf[56])
            if buf[63]:
                spans["fsel_bounds_seen"] = (buf[63], buf[63])
        if buf[57]:
            spans["fin_counts_to_gather"] = (buf[57], buf[58] or buf[57])
            spans["fin_select"] = (buf[58] or buf[57], buf[59] or buf[57])
            spans["fin_emit"] = (buf[59] or buf[57], buf[60] or buf[57])
        counts = {"fin_listed": int(buf[61]), "fin_fallback": int(buf[62])} if buf[57] else {}
        for nm, base in (("fin_fastsel", 24), ("bracket_fastsel", 32)):
            st = [buf[base + i] for i in range(8) if buf[base + i]]
            if st:
                counts[nm + "_phase_us"] = [round((b - a) / 1e3, 2) for a, b in zip(st, st[1:])]
        out = {k: (round((a - t0) / 1e3, 2), round((b - t0) / 1e3, 2)) for k, (a, b) in
               sorted(spans.items(), key=lambda t: t[1][0])}
        out.update(counts)
        probes = {i: round((buf[i] - t0) / 1e3, 2) for i in range(64, 96) if buf[i]}
        if probes:
            out["probes_us"] = probes  # ad hoc phase probes (g_ktrace[64..95])
        return out

    def profile_read(self) -> dict:
        """{stage: (total_ms, intervals)} since the last read (syncs)."""
        n = len(L.STAGES)
        ms = (C.c_double * n)()
        cnt = (C.c_int64 * n)()
        check(lib().hire_ctx_profile_read(self.h, ms, cnt, n))
        return {L.STAGES[i]: (ms[i], cnt[i]) for i in range(n) if cnt[i]}

    def __del__(self):
        if getattr(self, "h", None) and L._lib is not None:
            L._lib.hire_ctx_destroy(self.h)


_ctx_cache: dict = {}


def default_context() -> Context:
    dev = torch.cuda.current_device()
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    c = _ctx_cache.get(key)
    if c is None:
        c = _ctx_cache[key] = Context(dev)
    return c


def _x2d(x: torch.Tensor, d: int) -> torch.Tensor:
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if x.dtype != torch.float32 or not x.is_cuda:
        raise ValueError("x must be a CUDA float32 tensor [B, d]")
    if x.shape[1] != d:
        raise L.HireInvalidArgument(L.ERR_INVALID, f"x has dim {x.shape[1]} but the matrix has {d} rows")
    return x.contiguous()


class ScoreMatrix:
    """Device-resident dense matrix W [l, d] (== the reference's d x l Z)."""

    def __init__(self, w: torch.Tensor, _handle=None, _parent=None):
        if w.dim() != 2 or not w.is_cuda:
            raise ValueError("ScoreMatrix needs a 2-D CUDA tensor [l, d]")
        if w.dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("ScoreMatrix dtype must be float32 or bfloat16")
        self.tensor = w.contiguous()
        self.rows, self.d = self.tensor.shape
        self.dtype = L.BF16 if self.tensor.dtype == torch.bfloat16 else L.F32
        self._parent = _parent
        if _handle is None:
            h = C.c_void_p()
            check(lib().hire_matrix_view(_ptr(self.tensor), self.rows, self.d, self.dtype, C.byref(h)))
            _handle = h
        self.h = _handle

    def slice_cols(self, first: int, count: int) -> "ScoreMatrix":
        h = C.c_void_p()
        check(lib().hire_matrix_slice(self.h, first, count, C.byref(h)))
        return ScoreMatrix(self.tensor[first:first + count], _handle=h, _parent=self)

    def __del__(self):
        if getattr(self, "h", None) and L._lib is not None:
            L._lib.hire_matrix_destroy(self.h)


class ApproxScorer:
    """The cheap proxy (approx.hpp:327): int4 per-row (HiRE-Q) or low-rank (HiRE-LR)."""

    def __init__(self, handle, kind, rows, d, rank=0, keep=()):
        self.h, self.kind, self.rows, self.d, self.rank = handle, kind, rows, d, rank
        self._keep = keep

    # approx.hpp:336 quantized(QuantizedMatrix)
    @staticmethod
    def quantized(codes: np.ndarray, scales: np.ndarray) -> "ApproxScorer":
        codes = np.ascontiguousarray(codes, dtype=np.int8)
        scales = np.ascontiguousarray(scales, dtype=np.float32)
        rows, d = codes.shape
        h = C.c_void_p()
        check(lib().hire_scorer_create_q4_codes(codes.ctypes.data_as(C.c_void_p),
                                                scales.ctypes.data_as(C.c_void_p), rows, d,
                                                C.byref(h)))
        return ApproxScorer(h, L.SCORER_Q4, rows, d)

    # HIRQ payload (approx.hpp:551-564)
    @staticmethod
    def from_hirq(payload: np.ndarray, scales: np.ndarray, rows: int, d: int) -> "ApproxScorer":
        payload = np.ascontiguousarray(payload, dtype=np.uint8)
        scales = np.ascontiguousarray(scales, dtype=np.float32)
        h = C.c_void_p()
        check(lib().hire_scorer_create_q4_hirq(payload.ctypes.data_as(C.c_void_p),
                                               scales.ctypes.data_as(C.c_void_p), rows, d,
                                               C.byref(h)))
        return ApproxScorer(h, L.SCORER_Q4, rows, d)

    # approx.hpp:342-347 low_rank_quantized(LowRankApprox): both factors
    # quantized per the int4 rule (per reference column: z1's d-vectors, z2's
    # l-vectors), scored over the dequantized entries code * scale — the
    # reference's own arithmetic (approx.hpp:500-516), so the strict low-rank
    # kernels reproduce it bit for bit. The int4 rule runs on the device (K9).
    @staticmethod
    def low_rank_quantized(z1: torch.Tensor, z2: torch.Tensor) -> "ApproxScorer":
        def q4_dequant(rows_major: torch.Tensor) -> np.ndarray:
            q = ApproxScorer.quantize(ScoreMatrix(rows_major.float().contiguous()))
            codes, scales = q.export_q4()
            return codes.astype(np.float32) * scales[:, None]   # fp32 code * scale, as entry()
        d1 = q4_dequant(z1)                                      # [r][d]: one row per z1 column
        d2 = np.ascontiguousarray(q4_dequant(z2.t()).T)          # z2 columns are [r] rows of z2^T
        a = ApproxScorer.low_rank(torch.from_numpy(d1).to(z1.device), torch.from_numpy(d2).to(z1.device))
        return a

    # approx.hpp:339 quantized(const ScoreMatrix&) — quantize_int4 on the device (K9)
    @staticmethod
    def quantize(z: ScoreMatrix, ctx: Optional[Context] = None) -> "ApproxScorer":
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib().hire_scorer_quantize(ctx.h, z.h, C.byref(h)))
        return ApproxScorer(h, L.SCORER_Q4, z.rows, z.d)

    # approx.hpp:332 low_rank(LowRankApprox): z1 [r, d], z2 [l, r] on the device
    @staticmethod
    def low_rank(z1: torch.Tensor, z2: torch.Tensor) -> "ApproxScorer":
        if z1.dtype != z2.dtype or z1.dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("low-rank factors must share dtype float32/bfloat16")
        r, d = z1.shape
        rows, r2 = z2.shape
        if r2 != r:
            raise L.HireInvalidArgument(L.ERR_INVALID, f"ApproxScorer: low-rank factors do not match rank {r}")
        dt = L.BF16 if z1.dtype == torch.bfloat16 else L.F32
        z1c, z2c = z1.contiguous(), z2.contiguous()
        h = C.c_void_p()
        check(lib().hire_scorer_create_lowrank(_ptr(z1c), _ptr(z2c), d, rows, r, dt, 1, C.byref(h)))
        return ApproxScorer(h, L.SCORER_LOWRANK, rows, d, r)

    def slice_cols(self, first: int, count: int) -> "ApproxScorer":
        h = C.c_void_p()
        check(lib().hire_scorer_slice(self.h, first, count, C.byref(h)))
        return ApproxScorer(h, self.kind, count, self.d, self.rank, keep=(self,))

    def input_dim(self) -> int:
        return self.d

    def output_dim(self) -> int:
        return self.rows

    def export_q4(self):
        codes = np.empty((self.rows, self.d), dtype=np.int8)
        scales = np.empty(self.rows, dtype=np.float32)
        check(lib().hire_scorer_export_q4(self.h, codes.ctypes.data_as(C.c_void_p),
                                          scales.ctypes.data_as(C.c_void_p)))
        return codes, scales

    # approx.hpp:382 scores(x, phi), batched
    def scores(self, x: torch.Tensor, phi="identity", x_mode: int = L.X_FP32, strict: bool = False,
               ctx: Optional[Context] = None) -> torch.Tensor:
        ctx = ctx or default_context()
        x = _x2d(x, self.d)
        out = torch.empty(x.shape[0], self.rows, dtype=torch.float32, device=x.device)
        check(lib().hire_scores(ctx.h, self.h, _ptr(x), x.shape[0], _phi(phi), x_mode, int(strict), _ptr(out)))
        return out

    def __del__(self):
        if getattr(self, "h", None) and L._lib is not None:
            L._lib.hire_scorer_destroy(self.h)


@dataclass
class HireConfig:
    """hire.hpp:16-20 plus the B200 knobs (see hire_topk_params)."""
    k: int = 1
    k_prime: int = 1
    phi: object = "identity"
    x_mode: int = L.X_FP32
    select: int = L.SELECT_EXACT
    strict: bool = False
    n_buckets: int = 0
    bucket_t: int = 0

    def params(self) -> L.TopkParams:
        return L.TopkParams(self.k, self.k_prime, _phi(self.phi), self.x_mode, self.select,
                            int(self.strict), self.n_buckets, self.bucket_t)


@dataclass
class HireResult:
    """hire.hpp:41-44: top-k (rank order) and the candidate set (ascending)."""
    top_idx: torch.Tensor   # [B, n_top] int32
    top_val: torch.Tensor   # [B, n_top] float32, exact against Z
    cand: Optional[torch.Tensor]  # [B, n_cand] int32 ascending
    clamped: bool
    top_prob: Optional[torch.Tensor] = None


def hire_topk(x: torch.Tensor, z: ScoreMatrix, a: ApproxScorer, cfg: HireConfig,
              ctx: Optional[Context] = None, want_candidates: bool = True,
              _probs: bool = False) -> HireResult:
    """hire.hpp:50-86 for a batch of queries."""
    ctx = ctx or default_context()
    x = _x2d(x, z.d)
    B = x.shape[0]
    cand = torch.empty(B, max(cfg.k_prime, 1), dtype=torch.int32, device=x.device) if want_candidates else None
    kk = max(cfg.k, 1)
    ti = torch.empty(B, kk, dtype=torch.int32, device=x.device)
    tv = torch.empty(B, kk, dtype=torch.float32, device=x.device)
    tp = torch.empty(B, kk, dtype=torch.float32, device=x.device) if _probs else None
    nc, nt, cl = C.c_int64(), C.c_int64(), C.c_int()
    p = cfg.params()
    check(lib().hire_topk_run(ctx.h, z.h, a.h, _ptr(x), B, C.byref(p), _ptr(cand), _ptr(ti), _ptr(tv),
                              _ptr(tp), C.byref(nc), C.byref(nt), C.byref(cl)))
    return HireResult(ti[:, :nt.value], tv[:, :nt.value],
                      cand[:, :nc.value] if cand is not None else None, bool(cl.value),
                      tp[:, :nt.value] if tp is not None else None)


def softmax_topk(w: ScoreMatrix, x: torch.Tensor, a: ApproxScorer, cfg: HireConfig,
                 ctx: Optional[Context] = None):
    """hire.hpp:123-144: (indices [B,k] by probability desc, probabilities)."""
    if _phi(cfg.phi) != 0:
        raise L.HireInvalidArgument(L.ERR_INVALID, "softmax_topk: phi must be identity")
    r = hire_topk(x, w, a, cfg, ctx, want_candidates=False, _probs=True)
    return r.top_idx, r.top_prob


def matvec(z: ScoreMatrix, x: torch.Tensor, phi="identity", strict: bool = False,
           ctx: Optional[Context] = None) -> torch.Tensor:
    """linalg.hpp:148-154 (batched). Shares the exact-recompute reduction."""
    ctx = ctx or default_context()
    x = _x2d(x, z.d)
    out = torch.empty(x.shape[0], z.rows, dtype=torch.float32, device=x.device)
    check(lib().hire_matvec(ctx.h, z.h, _ptr(x), x.shape[0], _phi(phi), int(strict), _ptr(out)))
    return out


def topk_select(v: torch.Tensor, k: int, ctx: Optional[Context] = None):
    """linalg.hpp:157-176 on each row of v [B, n]: (idx, val, clamped)."""
    ctx = ctx or default_context()
    if v.dim() == 1:
        v = v.unsqueeze(0)
    v = v.contiguous().float()
    B, n = v.shape
    kk = min(k, n) if k >= 1 else 1
    idx = torch.empty(B, kk, dtype=torch.int32, device=v.device)
    val = torch.empty(B, kk, dtype=torch.float32, device=v.device)
    cl = C.c_int()
    check(lib().hire_topk_select(ctx.h, _ptr(v), B, n, k, _ptr(idx), _ptr(val), C.byref(cl)))
    return idx, val, bool(cl.value)


def exact_topk(z: ScoreMatrix, x: torch.Tensor, k: int, phi="identity", strict: bool = False,
               ctx: Optional[Context] = None):
    """linalg.hpp:184-188."""
    return topk_select(matvec(z, x, phi, strict, ctx), k, ctx)


@dataclass
class GroupedFFN:
    """ffn.hpp:19-28: U, V [m, d] (the reference's d x m), group size, phi."""
    u: ScoreMatrix
    v: ScoreMatrix
    group_size: int = 1
    phi: object = "relu"

    def dim(self) -> int:
        return self.u.d

    def hidden(self) -> int:
        return self.u.rows


def ffn_group_sparse(f: GroupedFFN, x: torch.Tensor, a: ApproxScorer, k: int, k_prime: int,
                     x_mode: int = L.X_FP32, strict: bool = False, ctx: Optional[Context] = None):
    """ffn.hpp:211-219: (output [B, d], selected group ids [B, k/g] ascending)."""
    ctx = ctx or default_context()
    x = _x2d(x, f.u.d)
    B = x.shape[0]
    g = f.group_size
    sel = torch.empty(B, max(k // max(g, 1), 1), dtype=torch.int32, device=x.device)
    out = torch.empty(B, f.u.d, dtype=torch.float32, device=x.device)
    p = L.FfnParams(k, k_prime, g, _phi(f.phi), x_mode, int(strict), 0)
    check(lib().hire_ffn_run(ctx.h, f.u.h, f.v.h, a.h, _ptr(x), B, C.byref(p), _ptr(sel), _ptr(out)))
    return out, sel


def ffn_dense(f: GroupedFFN, x: torch.Tensor, strict: bool = False, ctx: Optional[Context] = None):
    """ffn.hpp:65-76."""
    ctx = ctx or default_context()
    x = _x2d(x, f.u.d)
    out = torch.empty(x.shape[0], f.u.d, dtype=torch.float32, device=x.device)
    check(lib().hire_ffn_dense_run(ctx.h, f.u.h, f.v.h, _ptr(x), x.shape[0], _phi(f.phi), int(strict), _ptr(out)))
    return out


def union_group_select(f: GroupedFFN, xs: torch.Tensor, a: ApproxScorer, k: int, k_prime: int,
                       x_mode: int = L.X_FP32, strict: bool = False, ctx: Optional[Context] = None) -> np.ndarray:
    """ffn.hpp:237-253: sorted union of the per-sample select_groups results
    (the paper's dynamic overlap across a batch)."""
    ctx = ctx or default_context()
    xs = _x2d(xs, f.u.d)
    g = f.group_size
    ids = torch.empty(max(f.u.rows // max(g, 1), 1), dtype=torch.int32, device=xs.device)
    n = C.c_int64()
    p = L.FfnParams(k, k_prime, g, _phi(f.phi), x_mode, int(strict), 0)
    check(lib().hire_ffn_union_select(ctx.h, f.u.h, a.h, _ptr(xs), xs.shape[0], C.byref(p), _ptr(ids), C.byref(n)))
    return ids[:n.value].cpu().numpy().astype(np.uint32)


@dataclass
class CommonPathFFN:
    """ffn.hpp:44-47: a dense part (every unit, every token) plus a
    group-sparse part; `dense_part` None = no dense units."""
    dense_part: Optional[GroupedFFN]
    sparse_part: GroupedFFN


def ffn_common_path(c: CommonPathFFN, x: torch.Tensor, a: ApproxScorer, k: int, k_prime: int,
                    x_mode: int = L.X_FP32, strict: bool = False, ctx: Optional[Context] = None) -> torch.Tensor:
    """ffn.hpp:223-234: ffn_dense(dense part) + ffn_group_sparse(sparse part)."""
    ctx = ctx or default_context()
    sp = c.sparse_part
    x = _x2d(x, sp.u.d)
    out = torch.empty(x.shape[0], sp.u.d, dtype=torch.float32, device=x.device)
    p = L.FfnParams(k, k_prime, sp.group_size, _phi(sp.phi), x_mode, int(strict), 0)
    du = c.dense_part.u.h if c.dense_part is not None else None
    dv = c.dense_part.v.h if c.dense_part is not None else None
    check(lib().hire_ffn_common_path_run(ctx.h, du, dv, sp.u.h, sp.v.h, a.h, _ptr(x), x.shape[0], C.byref(p),
                                         _ptr(out)))
    return out


def overlap_ratio(per_sample_sets, k_groups: int) -> float:
    """metrics.hpp:68-88: |union| / (s * k_groups); 1/s when every sample
    selects the same groups, 1 when the selections are disjoint."""
    if len(per_sample_sets) == 0:
        raise L.HireInvalidArgument(L.ERR_INVALID, "overlap_ratio: no sample sets")
    if k_groups < 1:
        raise L.HireInvalidArgument(L.ERR_INVALID, "overlap_ratio: k_groups must be >= 1")
    merged = set()
    for s_ in per_sample_sets:
        if len(s_) != k_groups:
            raise L.HireInvalidArgument(L.ERR_INVALID,
                                        f"overlap_ratio: sample selected {len(s_)} groups, expected {k_groups}")
        merged.update(int(v) for v in s_)
    return len(merged) / (len(per_sample_sets) * k_groups)


def shard_range(l: int, s: int, i: int):
    """distributed.hpp:53-57: (first, width) of shard i of s."""
    base, extra = divmod(l, s)
    return i * base + min(i, extra), base + (1 if i < extra else 0)


def da_topk_emulated(z: ScoreMatrix, a: ApproxScorer, x: torch.Tensor, s: int, cfg: HireConfig,
                     merge: int = L.MERGE_PER_SHARD, uneven: bool = False,
                     ctx: Optional[Context] = None):
    """distributed.hpp:73-134 with all s shards on this GPU (no collective)."""
    ctx = ctx or default_context()
    x = _x2d(x, z.d)
    B = x.shape[0]
    cap = max(cfg.k, 1)
    ti = torch.empty(B, cap, dtype=torch.int32, device=x.device)
    tv = torch.empty(B, cap, dtype=torch.float32, device=x.device)
    n, cl = C.c_int64(), C.c_int()
    p = cfg.params()
    check(lib().hire_da_topk_emulated(ctx.h, z.h, a.h, s, _ptr(x), B, C.byref(p), merge, int(uneven),
                                      _ptr(ti), _ptr(tv), C.byref(n), C.byref(cl)))
    return ti[:, :n.value], tv[:, :n.value], bool(cl.value)


def da_group_sparse_emulated(f: GroupedFFN, x: torch.Tensor, a: ApproxScorer, k: int, k_prime: int,
                             s: int, x_mode: int = L.X_FP32, strict: bool = False,
                             uneven: bool = False, ctx: Optional[Context] = None):
    """distributed.hpp:145-206 with all s shards on this GPU."""
    ctx = ctx or default_context()
    x = _x2d(x, f.u.d)
    B = x.shape[0]
    g = f.group_size
    sel = torch.empty(B, max(k // max(g, 1), 1), dtype=torch.int32, device=x.device)
    out = torch.empty(B, f.u.d, dtype=torch.float32, device=x.device)
    p = L.FfnParams(k, k_prime, g, _phi(f.phi), x_mode, int(strict), 0)
    check(lib().hire_da_ffn_emulated(ctx.h, f.u.h, f.v.h, a.h, s, _ptr(x), B, C.byref(p), int(uneven),
                                     _ptr(sel), _ptr(out)))
    return out, sel


@dataclass
class CostReport:
    """metrics.hpp:43-51."""
    bytes_baseline: int = 0
    bytes_lr: int = 0
    bytes_q: int = 0
    bytes_lrq: int = 0
    lr_no_saving: bool = False
    q_no_saving: bool = False
    lrq_no_saving: bool = False


def param_bytes(d: int, l: int, r: int, k_prime: int) -> CostReport:
    """metrics.hpp:51-64: the paper's parameter bytes per query (bf16 dense
    2dl; low-rank 2(dr + rl + dk'); int4 ceil(dl/2) + 2dk'; LRQ
    ceil((dr + rl)/2) + 2dk'). Like the reference it omits the int4 scales;
    roofline_bytes adds them."""
    if d < 1 or l < 1 or r < 1:
        raise L.HireInvalidArgument(L.ERR_INVALID, "param_bytes: dims must be positive")
    c = CostReport()
    c.bytes_baseline = 2 * d * l
    c.bytes_lr = 2 * (d * r + r * l + d * k_prime)
    c.bytes_q = (d * l + 1) // 2 + 2 * d * k_prime
    c.bytes_lrq = (d * r + r * l + 1) // 2 + 2 * d * k_prime
    c.lr_no_saving = c.bytes_lr >= c.bytes_baseline
    c.q_no_saving = c.bytes_q >= c.bytes_baseline
    c.lrq_no_saving = c.bytes_lrq >= c.bytes_baseline
    return c


def roofline_bytes(proxy: str, d: int, l: int, gathered_rows: int, row_bytes: int, r: int = 0,
                   factor_bytes: int = 2, extra_rows: int = 0, exchange_bytes: int = 0) -> int:
    """HBM bytes one step must move:
    proxy bytes INCLUDING the int4 scales (param_bytes' Q term omits them)
    + unique gathered rows x row bytes (+ extra_rows: the FFN's V rows)
    + all-gather bytes. proxy 'q4': ceil(dl/2) + 4l; 'lowrank': (dr + rl) x
    factor_bytes. gathered_rows counts each row once per step (batch union)."""
    if proxy == "q4":
        pb = (d * l + 1) // 2 + 4 * l
    elif proxy == "lowrank":
        pb = (d * r + r * l) * factor_bytes
    else:
        raise ValueError(f"unknown proxy kind {proxy!r}")
    return pb + (gathered_rows + extra_rows) * row_bytes + exchange_bytes


@dataclass
class GatherBenchConfig:
    """gather_bench.hpp:18-25."""
    n_groups: int = 4096
    g: int = 8
    d: int = 128
    fraction_selected: float = 0.25
    repeats: int = 9
    seed: int = 0


@dataclass
class GatherBenchResult:
    """gather_bench.hpp:38-46 (times in ns, CUDA events, device memory)."""
    sparse_ns: float
    dense_ns: float
    efficiency_paper: float
    efficiency_ratio: float
    bytes_moved: int
    groups_selected: int
    checksum_ok: bool


def run_gather_bench(cfg: GatherBenchConfig, ctx: Optional[Context] = None) -> GatherBenchResult:
    """run_gather_bench (gather_bench.hpp:71-152) on the GPU: gather a seeded
    random subset of groups (the reference's Fisher-Yates selection, draw
    order) vs a dense copy of the same bytes; the paper's group-size argument
    (contiguous groups of g rows gather near dense bandwidth)."""
    ctx = ctx or default_context()
    c = L.GatherBenchConfig(cfg.n_groups, cfg.g, cfg.d, cfg.fraction_selected, cfg.repeats, cfg.seed)
    r = L.GatherBenchResult()
    check(lib().hire_gather_bench(ctx.h, C.byref(c), C.byref(r)))
    return GatherBenchResult(r.sparse_ns, r.dense_ns, r.efficiency_paper, r.efficiency_ratio, r.bytes_moved,
                             r.groups_selected, bool(r.checksum_ok))


def recall(cand: np.ndarray, exact_idx: np.ndarray):
    """metrics.hpp:23-34 for one query: (recall, intersection_k, top1_agree)."""
    cand = np.asarray(cand)
    exact_idx = np.asarray(exact_idx)
    if exact_idx.size == 0:
        return 0.0, 0, False
    hit = np.isin(exact_idx, cand)
    return float(hit.mean()), int(hit.sum()), bool(hit[0])
