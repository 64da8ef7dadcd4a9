"""DA-TOP-k across GPUs: one process per GPU, NCCL over NVLink/NVSwitch.

Reference: distributed.hpp:41-63 (shard), :73-134 (da_topk), :145-206
(da_group_sparse). The reference simulates shards in one process and
concatenates in memory; here every rank owns the rows [first, first+width)
of the width rule, runs the local stage on its GPU, and the per-shard
(score, global index) pairs travel as 8-byte rank keys through one
ncclAllGather inside hire_da_topk_run (the FFN's selected ids and partial
outputs through one grouped all-gather inside hire_da_ffn_run, summed in
rank order). The two halves of each call (`*_local`: this rank's keys /
partials into a device buffer; `*_merge`: the gathered buffer into the
result) are exposed too, for callers that move the bytes themselves.

The host-side rules (partition, quotas, key encoding, merge) are also
exposed as plain functions so the multi-rank exchange can be exercised with
the gloo backend on CPU (tests/test_parallel_gloo.py).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _lib as L
from ._lib import check, lib
from .api import Context, GroupedFFN, HireConfig, ScoreMatrix, ApproxScorer, _phi, _ptr, _x2d, default_context


# ----------------------------------------------------------- host rules ---
def shard_range(l: int, s: int, i: int):
    """distributed.hpp:53-57: shard i of s covers [first, first+width)."""
    base, extra = divmod(l, s)
    return i * base + min(i, extra), base + (1 if i < extra else 0)


def quota(k: int, s: int, i: int) -> int:
    """Per-shard quota. The reference requires s | k (distributed.hpp:79-85);
    for s not dividing k the first k % s shards take one more."""
    return k // s + (1 if i < k % s else 0)


def check_divisible(k: int, k_prime: int, s: int, uneven: bool) -> None:
    if uneven:
        return
    if k % s:
        raise L.HireInvalidArgument(L.ERR_INVALID, f"da_topk: s = {s} must divide k = {k}")
    if k_prime % s:
        raise L.HireInvalidArgument(L.ERR_INVALID, f"da_topk: s = {s} must divide k_prime = {k_prime}")


def encode_keys(values: np.ndarray, indices: np.ndarray) -> np.ndarray:
    """(value, index) -> u64 rank key, larger = ranks first (linalg.hpp:129-133).
    Same encoding as csrc/common.cuh make_key; -0.0 ranks equal to +0.0."""
    v = np.ascontiguousarray(values, dtype=np.float32).copy()
    u = v.view(np.uint32).copy()
    u[u == 0x80000000] = 0
    neg = (u & 0x80000000) != 0
    o = np.where(neg, ~u, u | np.uint32(0x80000000)).astype(np.uint64)
    idx = np.asarray(indices, dtype=np.uint64)
    return (o << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - idx)


def decode_keys(keys: np.ndarray):
    k = np.asarray(keys, dtype=np.uint64)
    o = (k >> np.uint64(32)).astype(np.uint32)
    u = np.where((o & 0x80000000) != 0, o & np.uint32(0x7FFFFFFF), ~o).astype(np.uint32)
    idx = (np.uint64(0xFFFFFFFF) - (k & np.uint64(0xFFFFFFFF))).astype(np.uint32)
    return u.view(np.float32), idx


def merge_gathered(gathered: np.ndarray, K: int):
    """The device merge (final_select_kernel) restated on the host: the K
    largest non-padding keys of the gathered [D, n_per] buffer, rank order."""
    flat = np.asarray(gathered, dtype=np.uint64).reshape(-1)
    flat = flat[flat != 0]
    top = np.sort(flat)[::-1][:K]
    return decode_keys(top)


# ------------------------------------------------------------ NCCL path ---
class Communicator:
    """hire_comm over NCCL; the unique id is broadcast with torch.distributed
    (whatever backend the process group uses)."""

    def __init__(self, world: int, rank: int, group=None):
        import torch.distributed as dist
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            check(lib().hire_comm_unique_id(uid))
        obj = [bytes(uid)] if rank == 0 else [None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        buf = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        check(lib().hire_comm_create(buf, world, rank, C.byref(h)))
        self.h, self.world, self.rank = h, world, rank

    def __del__(self):
        if getattr(self, "h", None) and L._lib is not None:
            L._lib.hire_comm_destroy(self.h)


def da_topk(z_shard: ScoreMatrix, a_shard: ApproxScorer, total_rows: int, x: torch.Tensor,
            cfg: HireConfig, comm: Optional[Communicator], merge: int = L.MERGE_PER_SHARD,
            uneven: bool = False, ctx: Optional[Context] = None):
    """This rank's call of DA-TOP-k; returns the merged (idx, val, clamped) on every rank."""
    ctx = ctx or default_context()
    world = comm.world if comm else 1
    rank = comm.rank if comm else 0
    x = _x2d(x, z_shard.d)
    B = x.shape[0]
    cap = max(cfg.k, 1)
    ti = torch.empty(B, cap, dtype=torch.int32, device=x.device)
    tv = torch.empty(B, cap, dtype=torch.float32, device=x.device)
    n, cl = C.c_int64(), C.c_int()
    p = cfg.params()
    check(lib().hire_da_topk_run(ctx.h, comm.h if comm else None, z_shard.h, a_shard.h, total_rows,
                                 world, rank, _ptr(x), B, C.byref(p), merge, int(uneven), _ptr(ti),
                                 _ptr(tv), C.byref(n), C.byref(cl)))
    return ti[:, :n.value], tv[:, :n.value], bool(cl.value)


def da_group_sparse(f_shard: GroupedFFN, a_shard: ApproxScorer, total_units: int, x: torch.Tensor,
                    k: int, k_prime: int, comm: Optional[Communicator], x_mode: int = L.X_FP32,
                    uneven: bool = False, ctx: Optional[Context] = None):
    """This rank's call of da_group_sparse: (out [B,d] summed over ranks, union of groups)."""
    ctx = ctx or default_context()
    world = comm.world if comm else 1
    rank = comm.rank if comm else 0
    x = _x2d(x, f_shard.u.d)
    B = x.shape[0]
    g = f_shard.group_size
    sel = torch.empty(B, max(k // g, 1), dtype=torch.int32, device=x.device)
    out = torch.empty(B, f_shard.u.d, dtype=torch.float32, device=x.device)
    p = L.FfnParams(k, k_prime, g, _phi(f_shard.phi), x_mode, 0, 0)
    check(lib().hire_da_ffn_run(ctx.h, comm.h if comm else None, f_shard.u.h, f_shard.v.h, a_shard.h,
                                total_units, world, rank, _ptr(x), B, C.byref(p), int(uneven),
                                _ptr(sel), _ptr(out)))
    return out, sel


# ------------------------------------------------- local / merge halves ---
def da_topk_slots(cfg: HireConfig, world: int, merge: int = L.MERGE_PER_SHARD) -> int:
    n = C.c_int64()
    p = cfg.params()
    check(lib().hire_da_topk_slots(C.byref(p), world, merge, C.byref(n)))
    return n.value


def da_topk_local(z_shard: ScoreMatrix, a_shard: ApproxScorer, total_rows: int, world: int, rank: int,
                  x: torch.Tensor, cfg: HireConfig, merge: int = L.MERGE_PER_SHARD, uneven: bool = False,
                  ctx: Optional[Context] = None) -> torch.Tensor:
    """This rank's local stage (distributed.hpp:94-125): int64 view of the
    u64 rank keys [B, slots] (global indices; padding 0)."""
    ctx = ctx or default_context()
    x = _x2d(x, z_shard.d)
    B = x.shape[0]
    send = torch.zeros(B, da_topk_slots(cfg, world, merge), dtype=torch.int64, device=x.device)
    p = cfg.params()
    check(lib().hire_da_topk_local(ctx.h, z_shard.h, a_shard.h, total_rows, world, rank, _ptr(x), B, C.byref(p),
                                   merge, int(uneven), _ptr(send)))
    return send


def da_topk_merge(gathered: torch.Tensor, total_rows: int, world: int, cfg: HireConfig,
                  merge: int = L.MERGE_PER_SHARD, uneven: bool = False, ctx: Optional[Context] = None):
    """Merge of the gathered keys [world, B, slots] (distributed.hpp:127-131):
    (idx, val, clamped), identical on every rank."""
    ctx = ctx or default_context()
    g = gathered.contiguous()
    B = g.shape[1]
    cap = max(cfg.k, 1)
    ti = torch.empty(B, cap, dtype=torch.int32, device=g.device)
    tv = torch.empty(B, cap, dtype=torch.float32, device=g.device)
    n, cl = C.c_int64(), C.c_int()
    p = cfg.params()
    check(lib().hire_da_topk_merge(ctx.h, _ptr(g), total_rows, world, B, C.byref(p), merge, int(uneven),
                                   _ptr(ti), _ptr(tv), C.byref(n), C.byref(cl)))
    return ti[:, :n.value], tv[:, :n.value], bool(cl.value)


def _ffn_params(f: GroupedFFN, k: int, k_prime: int, x_mode: int, strict: bool = False):
    return L.FfnParams(k, k_prime, f.group_size, _phi(f.phi), x_mode, int(strict), 0)


def da_ffn_slots(k: int, group_size: int, world: int) -> int:
    n = C.c_int64()
    p = L.FfnParams(k, k, group_size, 0, 0, 0, 0)
    check(lib().hire_da_ffn_slots(C.byref(p), world, C.byref(n)))
    return n.value


def da_ffn_local(f_shard: GroupedFFN, a_shard: ApproxScorer, total_units: int, world: int, rank: int,
                 x: torch.Tensor, k: int, k_prime: int, x_mode: int = L.X_FP32, uneven: bool = False,
                 strict: bool = False, ctx: Optional[Context] = None):
    """This rank's local stage of da_group_sparse: (selected global group
    ids [B, slots] int32, partial output [B, d] fp32)."""
    ctx = ctx or default_context()
    x = _x2d(x, f_shard.u.d)
    B = x.shape[0]
    sel = torch.zeros(B, da_ffn_slots(k, f_shard.group_size, world), dtype=torch.int32, device=x.device)
    part = torch.empty(B, f_shard.u.d, dtype=torch.float32, device=x.device)
    p = _ffn_params(f_shard, k, k_prime, x_mode, strict)
    check(lib().hire_da_ffn_local(ctx.h, f_shard.u.h, f_shard.v.h, a_shard.h, total_units, world, rank, _ptr(x),
                                  B, C.byref(p), int(uneven), _ptr(sel), _ptr(part)))
    return sel, part


def da_ffn_merge(gathered_sel: torch.Tensor, gathered_parts: torch.Tensor, total_units: int, k: int,
                 group_size: int, uneven: bool = False, ctx: Optional[Context] = None):
    """Merge of the gathered ids [world, B, slots] and partials [world, B, d]:
    (out [B, d] = rank-order sum, union of groups [B, k/g])."""
    ctx = ctx or default_context()
    gs, gp = gathered_sel.contiguous(), gathered_parts.contiguous()
    world, B, d = gp.shape
    sel = torch.empty(B, max(k // group_size, 1), dtype=torch.int32, device=gp.device)
    out = torch.empty(B, d, dtype=torch.float32, device=gp.device)
    p = L.FfnParams(k, k, group_size, 0, 0, 0, 0)
    check(lib().hire_da_ffn_merge(ctx.h, _ptr(gs), _ptr(gp), total_units, d, world, B, C.byref(p), int(uneven),
                                  _ptr(sel), _ptr(out)))
    return out, sel
