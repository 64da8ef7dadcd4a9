#!/usr/bin/env python
"""HiRE approximate top-k path on B200 — benchmark (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload cfg3|cfg2|cfg1|cfg4|cfg5] [--batch B]

Default workload: BASELINE.json configs[2] (cfg3), the largest single-GPU
config — HiRE-softmax over V=256000, d=2048 (bf16 W, int4 per-row proxy
scored against int8-quantised x, exact top-k'=1024 candidates, gather
recompute, exact top-k=64 + softmax), batch 32 (configs[2] lists 1/8/32;
--batch picks another). A "step" is one call over one batch of decode
queries. Working set 1.3 GB > 126 MB L2, so every step streams from HBM.

N > 1 (`--gpus N`, re-executed under torchrun if not already launched by
it): DA-TOP-k strong scaling (distributed.hpp:73-134) — the same vocab and
batch, rows split across ranks by the width rule, each rank the local
stage on its shard, one ncclAllGather of (exact value, global index) keys,
global merge on every rank. --workload cfg4 is BASELINE's own DA config.

One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
_ADDR = {}


def _addr(a):
    """Address of a long-lived (pinned) numpy buffer, looked up once: numpy's
    `.ctypes.data` costs 1-2 us per access, a serving loop binds its buffers
    once ("per-call Python marshalling")."""
    k = id(a)
    v = _ADDR.get(k)
    if v is None or v[0] is not a:
        v = _ADDR[k] = (a, a.ctypes.data)
    return v[1]


METRIC = "HiRE decode tokens/s (µs/token, HBM roofline fraction, recall@k)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": PEAKS_FALLBACK["hbm_gbs"], "src": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------- dist utils --
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def da_path(world):
    """DA-TOP-k through hire_da_topk_run + NCCL: always at N > 1. HIRE_BENCH_DA=1
    takes the same code path on one GPU with a 1-rank communicator (validation
    of the N > 1 flow — graph capture of the ncclAllGather included — where
    only one GPU is available; not a bench configuration)."""
    return world > 1 or os.environ.get("HIRE_BENCH_DA") == "1"


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def relaunch_under_torchrun(n: int):
    """--gpus N without a torchrun parent: re-exec this script as N ranks."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execvp(cmd[0], cmd)


# ---------------------------------------------------------------- clocks ---
class ClockSampler:
    """Polls nvidia-smi (clocks + throttle reasons) from a thread while the
    timed region runs; bench.py also replays the same graph for a ~1 s soak
    right before the timed replay so the sample covers steady clocks."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int, period: float = 0.05):
        self.index, self.period = index, period
        self.rows = []

    def _poll(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout
                self.rows += [l for l in out.splitlines() if l.strip()]
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        import threading
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._poll, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm, mx, reasons = [], None, set()
        for l in self.rows:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "window": "1 s soak of the same graph + the timed replay"}


# ------------------------------------------------- weight generators (torch) --
# Plain torch on the device: used by both arms (the reference arm copies the
# result to the host; it never imports this repo's package).
def gen_ffn_layer(m, d, r, gen):
    """cfg2 family: N(0, 1/d) + 3 x a rank-r component with the same entry
    scale, bf16 (BASELINE.json configs[1])."""
    def one():
        base = torch.randn(m, d, device="cuda", generator=gen) / d ** 0.5
        A = torch.randn(m, r, device="cuda", generator=gen)
        Bm = torch.randn(r, d, device="cuda", generator=gen)
        return (base + 3.0 * (A @ Bm) / (r * d) ** 0.5).to(torch.bfloat16).contiguous()
    return one(), one()


def gen_vocab_rows(V, d, r, first, count, seed, lr_scale=1.0, noise=0.1, blk=4096):
    """Rows [first, first+count) of W [V, d] bf16 = lr_scale * A B / sqrt(r) +
    noise * N(0,1) (cfg3 / cfg4 family). Generated per 4096-row block from a
    per-block seed, so any shard of the width rule gets the same rows as the
    whole matrix (strong scaling compares like with like)."""
    gB = torch.Generator(device="cuda").manual_seed(seed)
    Bm = torch.randn(r, d, device="cuda", generator=gB)
    W = torch.empty(count, d, device="cuda", dtype=torch.bfloat16)
    A_out = torch.empty(count, r, device="cuda")
    for b0 in range(first // blk * blk, first + count, blk):
        g = torch.Generator(device="cuda").manual_seed(seed * 1_000_003 + b0 // blk + 1)
        n = min(blk, V - b0)
        A = torch.randn(n, r, device="cuda", generator=g)
        blkW = (lr_scale * (A @ Bm) / r ** 0.5 + noise * torch.randn(n, d, device="cuda", generator=g))
        s, e = max(first, b0), min(first + count, b0 + n)
        W[s - first:e - first] = blkW[s - b0:e - b0].to(torch.bfloat16)
        A_out[s - first:e - first] = A[s - b0:e - b0]
    return W, A_out, Bm


def shard_range(l, s, i):
    """distributed.hpp:53-57 (the same rule as parallel.shard_range)."""
    base, extra = divmod(l, s)
    return i * base + min(i, extra), base + (1 if i < extra else 0)


# -------------------------------------------------------------- workloads --
class Workload:
    """Shapes + torch weights; attach(H) builds the product's handles (our
    arm only); ref_host() returns host arrays for the reference arm."""
    name = ""
    lowrank = False
    dtype = "int4 x int8 -> int32 proxy, bf16 rows, fp32 accumulation"
    scaling = "weak"

    def query_scale(self):
        return 1.0 / np.sqrt(self.d)

    def inputs(self, n):
        return torch.randn(n, self.B, self.d, device="cuda", generator=self.gen) * float(self.query_scale())


class SoftmaxWorkload(Workload):
    """cfg3 (BASELINE.json configs[2]): HiRE-softmax, V=256000, d=2048, bf16
    W = rank-256 (unit entry variance) + 0.1 N(0,1), int4 per-row proxy
    (device K9) x int8 x, exact top-k'=1024, k=64, softmax over the top-k.
    N > 1: DA-TOP-k over the rows (global merge), strong scaling."""
    name = "cfg3"

    def __init__(self, batch, select="exact", world=1, rank=0, seed=0):
        self.V, self.d, self.kp, self.k, self.B = 256000, 2048, 1024, 64, batch
        self.world, self.rank, self.select = world, rank, select
        self.da = da_path(world)
        self.first, self.width = shard_range(self.V, world, rank)
        self.Wt, _, _ = gen_vocab_rows(self.V, self.d, 256, self.first, self.width, seed=1 + seed)
        self.gen = torch.Generator(device="cuda").manual_seed(seed + 99)
        self.scaling = "strong" if world > 1 else "weak"
        torch.cuda.synchronize()

    def attach(self, H):
        import paper_2402_09360_b200.parallel as P
        self.H, self.P = H, P
        self.W = H.ScoreMatrix(self.Wt)
        self.A = H.ApproxScorer.quantize(self.W)
        kw = dict(k=self.k, k_prime=self.kp, x_mode=H.X_INT8)
        if self.select == "bucketed":
            kw.update(select=H.SELECT_BUCKETED, n_buckets=1024, bucket_t=1)
        self.cfg = H.HireConfig(**kw)
        self.comm = P.Communicator(self.world, self.rank) if self.da else None
        torch.cuda.synchronize()

    @property
    def proxy_kernel(self):
        if self.B >= 5:
            return "q4_score_umma (K1 on tcgen05: TMA ring -> TMEM A operand -> kind::i8 MMA)"
        return "q4_score_mma_sel (K1F: IMMA proxy GEMV + fused candidate pre-selection)"

    def step(self, i, x):
        if self.da:
            return self.P.da_topk(self.W, self.A, self.V, x, self.cfg, self.comm, merge=self.H.MERGE_GLOBAL)
        # softmax_topk (hire.hpp:123-144): top-k indices + probabilities
        return self.H.softmax_topk(self.W, x, self.A, self.cfg)

    def host_step(self, i, x_host, idx_host, val_host, ctx):
        H = self.H
        if self.da:
            if not hasattr(self, "_xd"):
                self._xd = torch.empty(self.B, self.d, device="cuda")
            self._xd.copy_(torch.from_numpy(x_host), non_blocking=True)
            ti, tv, _ = self.P.da_topk(self.W, self.A, self.V, self._xd, self.cfg, self.comm,
                                       merge=H.MERGE_GLOBAL)
            torch.from_numpy(idx_host.view(np.int32)).copy_(ti, non_blocking=True)
            torch.from_numpy(val_host).copy_(tv, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return
        if not hasattr(self, "_hp"):  # call parameters built once, as a serving loop would
            self._hp = C.byref(self.cfg.params())
            self._hn = (C.c_int64(), C.c_int64(), C.c_int())
            self._hr = tuple(C.byref(v) for v in self._hn)
        # softmax_topk through the C ABI: top-k indices and probabilities
        H._lib.check(H.lib().hire_topk_host(ctx.h, self.W.h, self.A.h, _addr(x_host), self.B, self._hp, None,
                                            _addr(idx_host), _addr(self._hv), _addr(val_host),
                                            *self._hr))

    def host_buffers(self, pinned):
        self._hv = pinned((self.B, self.k), torch.float32)  # the exact values (not returned by softmax_topk)

    def io_bytes(self):
        return self.B * self.d * 4, self.B * self.k * 8

    def proxy_bytes(self):
        return self.width * (self.d // 2 + 4)

    def unique_rows(self, x):
        """unique candidate rows of this rank's shard over the batch (the
        gather kernel reads each once from HBM; repeats hit L2)."""
        kpl = self.P.quota(self.kp, self.world, self.rank)
        s = self.A.scores(x, x_mode=self.H.X_INT8)
        cand, _, _ = self.H.topk_select(s, kpl)
        return int(torch.unique(cand.long()).numel())

    def kernel_bytes(self, nu):
        return {"recompute": nu * self.d * 2}

    def step_bytes(self, x):
        nu = self.unique_rows(x)
        xb = self.world * self.B * (self.kp // self.world) * 8 if self.world > 1 else 0
        return self.H.roofline_bytes("q4", self.d, self.width, nu, self.d * 2, exchange_bytes=xb), nu, 0

    def recall(self, x):
        if self.da:
            return None
        H = self.H
        r = H.hire_topk(x, self.W, self.A, self.cfg)
        ex, _, _ = H.exact_topk(self.W, x, self.k)
        return float(np.mean([H.recall(r.cand[b].cpu().numpy(), ex[b].cpu().numpy())[0]
                              for b in range(x.shape[0])]))

    def config(self):
        return {"workload": "cfg3 HiRE-softmax (BASELINE.json configs[2])", "V": self.V, "d": self.d,
                "k_prime": self.kp, "k": self.k, "global_batch": self.B,
                "api": "softmax_topk (hire.hpp:123-144): top-k indices + softmax probabilities"
                       + (" via DA-TOP-k, global merge" if self.da else ""),
                "proxy": "int4 per-row absmax (device K9) x int8-quantised x",
                "weights": "bf16 W = rank-256 (unit entry variance) + 0.1 N(0,1)",
                "shard_rows": self.width,
                "l2": "working set 1.3 GB > 126 MB L2 (no flush needed)",
                "select": "1024 buckets x top-1 (literal)" if self.select == "bucketed" else "exact top-k'"}

    def ref_host(self):
        return {"W": self.Wt.float().cpu().numpy(), "quantize": True}


class FfnWorkload(Workload):
    """cfg2 (BASELINE.json configs[1]): one HiRE-FFN layer, d=2048, m=8192,
    bf16 U/V, int4 proxy of U x int8 x, k'=820, k=410, ReLU; 18 distinct
    layers cycled so every step streams cold weights from HBM."""
    name = "cfg2"

    def __init__(self, batch, layers=18, seed=0):
        self.m, self.d, self.kp, self.k, self.B = 8192, 2048, 820, 410, batch
        gen = torch.Generator(device="cuda").manual_seed(seed)
        self.uv = [gen_ffn_layer(self.m, self.d, 128, gen) for _ in range(layers)]
        self.gen = gen
        torch.cuda.synchronize()

    proxy_kernel = "q4_score_mma (K1 proxy GEMV, tensor-core IMMA)"

    def query_scale(self):
        return 1.0

    def attach(self, H):
        self.H = H
        self.layers = []
        for u, v in self.uv:
            U, Vm = H.ScoreMatrix(u), H.ScoreMatrix(v)
            self.layers.append((H.GroupedFFN(U, Vm, 1, "relu"), H.ApproxScorer.quantize(U)))
        torch.cuda.synchronize()

    def step(self, i, x):
        f, a = self.layers[i % len(self.layers)]
        return self.H.ffn_group_sparse(f, x, a, self.k, self.kp, x_mode=self.H.X_INT8)

    def host_step(self, i, x_host, sel_host, out_host, ctx):
        H = self.H
        f, a = self.layers[i % len(self.layers)]
        if not hasattr(self, "_hp"):
            self._hp = C.byref(H._lib.FfnParams(self.k, self.kp, 1, 1, H.X_INT8, 0, 0))
        H._lib.check(H.lib().hire_ffn_host(ctx.h, f.u.h, f.v.h, a.h, _addr(x_host), self.B, self._hp,
                                           _addr(sel_host), _addr(out_host)))

    def host_buffers(self, pinned):
        pass

    def io_bytes(self):
        return self.B * self.d * 4, self.B * self.k * 4 + self.B * self.d * 4

    def proxy_bytes(self):
        return self.m * (self.d // 2 + 4)

    def unique_rows(self, x):
        H = self.H
        f, a = self.layers[0]
        s = a.scores(x, phi="relu", x_mode=H.X_INT8)
        cand, _, _ = H.topk_select(s, self.kp)
        _, sel = H.ffn_group_sparse(f, x, a, self.k, self.kp, x_mode=H.X_INT8)
        return int(torch.unique(cand.long()).numel()), int(torch.unique(sel.long()).numel())

    def kernel_bytes(self, nu):
        return {"recompute": nu[0] * self.d * 2, "down": nu[1] * self.d * 2}

    def step_bytes(self, x):
        nu, nv = self.unique_rows(x)
        return self.H.roofline_bytes("q4", self.d, self.m, nu, self.d * 2, extra_rows=nv), (nu, nv), nv

    def recall(self, x):
        H = self.H
        f, a = self.layers[0]
        _, sel = H.ffn_group_sparse(f, x, a, self.k, self.kp, x_mode=H.X_INT8)
        ex, _, _ = H.exact_topk(f.u, x, self.k, "relu")
        return float(np.mean([H.recall(sel[b].cpu().numpy(), ex[b].cpu().numpy())[0] for b in range(x.shape[0])]))

    def config(self):
        return {"workload": "cfg2 HiRE-FFN layer (BASELINE.json configs[1])", "d": self.d,
                "m": self.m, "k_prime": self.kp, "k": self.k, "global_batch": self.B,
                "api": "ffn_group_sparse (ffn.hpp:211-219)",
                "proxy": "int4 per-row absmax (device K9) x int8-quantised x",
                "weights": "bf16 U,V = N(0,1/d) + 3x rank-128 (random init)",
                "l2": f"{len(self.uv)} distinct layers cycled (1.36 GB > 126 MB L2)",
                "select": "exact top-k' (topk_select)"}

    def ref_host(self):
        u, v = self.uv[0]
        return {"U": u.float().cpu().numpy(), "V": v.float().cpu().numpy(), "quantize": True}


class LowRankSoftmaxWorkload(Workload):
    """cfg1 (BASELINE.json configs[0]): HiRE-softmax, fp32, d=1024, V=32768,
    W = A B / 8 + 0.1 N(0,1), rank-64 truncated-SVD proxy, exact top-k'=256,
    k=32, batch 1. 16 copies cycled (9.7 MB working set per step)."""
    name = "cfg1"
    lowrank = True
    proxy_kernel = "lr_score_mma (K2 low-rank proxy, tensor-core HMMA with exact bf16 splits)"
    dtype = "fp32 (W, factors, x; fp32 accumulation)"

    def __init__(self, batch, copies=16, seed=0):
        self.V, self.d, self.r, self.kp, self.k, self.B = 32768, 1024, 64, 256, 32, batch
        gen = torch.Generator(device="cuda").manual_seed(seed)
        A = torch.randn(self.V, 64, device="cuda", generator=gen)
        Bm = torch.randn(64, self.d, device="cuda", generator=gen)
        self.Wt = (A @ Bm) / 8.0 + 0.1 * torch.randn(self.V, self.d, device="cuda", generator=gen)
        U, S, Vt = torch.linalg.svd(self.Wt.T.double(), full_matrices=False)
        self.z1 = (U[:, :self.r] * S[:self.r]).T.float().contiguous()
        self.z2 = Vt[:self.r].T.float().contiguous()
        self.ncopies = copies
        self.gen = gen
        torch.cuda.synchronize()

    def attach(self, H):
        self.H = H
        self.copies = [(H.ScoreMatrix(self.Wt.clone()), H.ApproxScorer.low_rank(self.z1.clone(), self.z2.clone()))
                       for _ in range(self.ncopies)]
        self.cfg = H.HireConfig(k=self.k, k_prime=self.kp)
        torch.cuda.synchronize()

    def step(self, i, x):
        z, a = self.copies[i % len(self.copies)]
        return self.H.softmax_topk(z, x, a, self.cfg)

    def host_step(self, i, x_host, idx_host, val_host, ctx):
        H = self.H
        z, a = self.copies[i % len(self.copies)]
        if not hasattr(self, "_hp"):
            self._hp = C.byref(self.cfg.params())
            self._hn = (C.c_int64(), C.c_int64(), C.c_int())
            self._hr = tuple(C.byref(v) for v in self._hn)
        H._lib.check(H.lib().hire_topk_host(ctx.h, z.h, a.h, _addr(x_host), self.B, self._hp, None,
                                            _addr(idx_host), _addr(self._hv), _addr(val_host),
                                            *self._hr))

    def host_buffers(self, pinned):
        self._hv = pinned((self.B, self.k), torch.float32)

    def io_bytes(self):
        return self.B * self.d * 4, self.B * self.k * 8

    def proxy_bytes(self):
        return (self.V + self.d) * self.r * 4

    def unique_rows(self, x):
        z, a = self.copies[0]
        r = self.H.hire_topk(x, z, a, self.cfg)
        return int(torch.unique(r.cand.long()).numel())

    def kernel_bytes(self, nu):
        return {"recompute": nu * self.d * 4}

    def step_bytes(self, x):
        nu = self.unique_rows(x)
        return self.H.roofline_bytes("lowrank", self.d, self.V, nu, self.d * 4, r=self.r, factor_bytes=4), nu, 0

    def recall(self, x):
        H = self.H
        z, a = self.copies[0]
        r = H.hire_topk(x, z, a, self.cfg)
        ex, _, _ = H.exact_topk(z, x, self.k)
        return float(np.mean([H.recall(r.cand[b].cpu().numpy(), ex[b].cpu().numpy())[0]
                              for b in range(x.shape[0])]))

    def config(self):
        return {"workload": "cfg1 HiRE-softmax fp32, rank-64 SVD proxy (BASELINE.json configs[0])",
                "V": self.V, "d": self.d, "rank": self.r, "k_prime": self.kp, "k": self.k,
                "global_batch": self.B, "api": "softmax_topk (hire.hpp:123-144)",
                "weights": "fp32 W = A B / 8 + 0.1 N(0,1), truncated SVD factors",
                "l2": f"{self.ncopies} copies cycled", "select": "exact top-k'"}

    def ref_host(self):
        return {"W": self.Wt.cpu().numpy(), "z1": self.z1.cpu().numpy(), "z2": self.z2.cpu().numpy()}


class DaSoftmaxWorkload(Workload):
    """cfg4 (BASELINE.json configs[3]): DA-TOP-k sharded softmax, bf16 W
    [256000, 4096] (rank-64 + 0.1 N(0,1)), rank-64 bf16 factors, B=16,
    k'=2048, k=128, global merge. Rank r holds its shard of the width rule;
    one ncclAllGather of B x k'/D keys per step. N=1: hire_topk (the s = 1
    equivalence)."""
    name = "cfg4"
    lowrank = True
    roof_stage = "recompute"
    roof_kernel = "recompute_fast<bf16, 16> (row-gather exact recompute, K4)"
    proxy_kernel = "lr_score_mma (K2 low-rank proxy, tensor-core HMMA, bf16 factors, fp32 acc)"
    dtype = "bf16 W and factors, fp32 x and accumulation"

    def __init__(self, batch, world=1, rank=0, seed=0):
        self.V, self.d, self.r, self.kp, self.k, self.B = 256000, 4096, 64, 2048, 128, batch
        self.world, self.rank = world, rank
        self.da = da_path(world)
        self.first, self.width = shard_range(self.V, world, rank)
        self.Wt, A, Bm = gen_vocab_rows(self.V, self.d, self.r, self.first, self.width, seed=4 + seed)
        self.z1 = (Bm / self.r ** 0.5).to(torch.bfloat16).contiguous()   # [r, d]
        self.z2 = A.to(torch.bfloat16).contiguous()                      # [width, r]
        self.gen = torch.Generator(device="cuda").manual_seed(seed + 99)
        self.scaling = "strong" if world > 1 else "weak"
        torch.cuda.synchronize()

    def attach(self, H):
        import paper_2402_09360_b200.parallel as P
        self.H, self.P = H, P
        self.W = H.ScoreMatrix(self.Wt)
        self.A = H.ApproxScorer.low_rank(self.z1, self.z2)
        self.cfg = H.HireConfig(k=self.k, k_prime=self.kp)
        self.comm = P.Communicator(self.world, self.rank) if self.da else None
        torch.cuda.synchronize()

    def step(self, i, x):
        if not self.da:
            return self.H.softmax_topk(self.W, x, self.A, self.cfg)
        return self.P.da_topk(self.W, self.A, self.V, x, self.cfg, self.comm, merge=self.H.MERGE_GLOBAL)

    def host_step(self, i, x_host, idx_host, val_host, ctx):
        H = self.H
        if not self.da:
            if not hasattr(self, "_hp"):
                self._hp = C.byref(self.cfg.params())
                self._hn = (C.c_int64(), C.c_int64(), C.c_int())
                self._hr = tuple(C.byref(v) for v in self._hn)
            H._lib.check(H.lib().hire_topk_host(ctx.h, self.W.h, self.A.h, _addr(x_host), self.B, self._hp,
                                                None, _addr(idx_host), _addr(self._hv),
                                                _addr(val_host), *self._hr))
            return
        if not hasattr(self, "_xd"):
            self._xd = torch.empty(self.B, self.d, device="cuda")
        self._xd.copy_(torch.from_numpy(x_host), non_blocking=True)
        ti, tv, _ = self.P.da_topk(self.W, self.A, self.V, self._xd, self.cfg, self.comm, merge=H.MERGE_GLOBAL)
        torch.from_numpy(idx_host.view(np.int32)).copy_(ti, non_blocking=True)
        torch.from_numpy(val_host).copy_(tv, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    def host_buffers(self, pinned):
        self._hv = pinned((self.B, self.k), torch.float32)

    def io_bytes(self):
        return self.B * self.d * 4, self.B * self.k * 8

    def proxy_bytes(self):
        return (self.width + self.d) * self.r * 2

    def unique_rows(self, x):
        s = self.A.scores(x)
        cand, _, _ = self.H.topk_select(s, self.P.quota(self.kp, self.world, self.rank))
        return int(torch.unique(cand.long()).numel())

    def kernel_bytes(self, nu):
        return {"recompute": nu * self.d * 2}

    def step_bytes(self, x):
        nu = self.unique_rows(x)
        xb = self.world * self.B * (self.kp // self.world) * 8 if self.world > 1 else 0
        return self.H.roofline_bytes("lowrank", self.d, self.width, nu, self.d * 2, r=self.r, factor_bytes=2,
                                     exchange_bytes=xb), nu, 0

    def recall(self, x):
        if self.da:
            return None
        H = self.H
        r = H.hire_topk(x, self.W, self.A, self.cfg)
        ex, _, _ = H.exact_topk(self.W, x, self.k)
        return float(np.mean([H.recall(r.cand[b].cpu().numpy(), ex[b].cpu().numpy())[0]
                              for b in range(x.shape[0])]))

    def config(self):
        return {"workload": "cfg4 DA-TOP-k sharded softmax (BASELINE.json configs[3])", "V": self.V,
                "d": self.d, "rank": self.r, "k_prime": self.kp, "k": self.k, "global_batch": self.B,
                "shard_rows": self.width, "merge": "global (all k' exact pairs all-gathered)",
                "api": "softmax_topk at N=1; da_topk (distributed.hpp:73-134) at N>1",
                "weights": "bf16 W = rank-64 (unit variance) + 0.1 N(0,1); proxy = generator factors",
                "l2": "W shard + proxy > 126 MB L2", "select": "exact top-k'/D per shard"}

    def ref_host(self):
        return {"W": self.Wt.float().cpu().numpy(), "z1": self.z1.float().cpu().numpy(),
                "z2": self.z2.float().cpu().numpy()}


class DecoderWorkload(Workload):
    """cfg5 (BASELINE.json configs[4]): greedy decode steps of the 18-layer
    ReLU decoder (d=2048, FFN 8192 as HiRE-FFN top-5% with the int4 proxy,
    16 heads over a 1024-token KV cache, V=256000 HiRE-softmax k'=1024 k=64).
    Each step feeds the previous step's tokens (true autoregressive chain);
    dense parts are library code (decoder.py)."""
    name = "cfg5"
    proxy_kernel = "q4_score_mma / q4_score_mma_sel / q4_score_umma (all int4 proxy launches: 18 FFN + vocab)"
    span_kernel = None

    def __init__(self, batch, world=1, rank=0, seed=0):
        self.B, self.seed, self.world, self.rank = batch, seed, world, rank
        # N > 1: FFN hidden units and vocabulary DA-sharded across the ranks
        # (BASELINE configs[4]); the batch is decoded once by all ranks
        self.scaling = "strong" if world > 1 else "weak"

    def attach(self, H):
        from paper_2402_09360_b200.decoder import DecoderConfig, HireDecoder
        self.H = H
        self.cfg = DecoderConfig()
        self.d, self.k, self.kp = self.cfg.d, self.cfg.vocab_k, self.cfg.vocab_k_prime
        comm = None
        if self.world > 1:
            import paper_2402_09360_b200.parallel as P
            comm = P.Communicator(self.world, self.rank)
        self.m = HireDecoder(self.cfg, self.B, seed=self.seed, comm=comm)
        g = torch.Generator(device="cuda").manual_seed(self.seed + 5)
        self.tok = torch.randint(0, self.cfg.vocab, (self.B,), device="cuda", generator=g)
        self.tok0 = self.tok.clone()
        torch.cuda.synchronize()

    def inputs(self, n):
        return [None] * n

    def step(self, i, x):
        nxt, _, _ = self.m.step(self.tok)
        self.tok.copy_(nxt)
        return nxt

    def host_step(self, i, x_host, idx_host, val_host, ctx):
        if not hasattr(self, "_hg"):
            self._tin = torch.zeros(self.B, dtype=torch.int64, device="cuda")
            self._pin_in = torch.zeros(self.B, dtype=torch.int64).pin_memory()
            self._pin_out = torch.zeros(self.B, self.k, dtype=torch.int32).pin_memory()
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                self.m.step(self._tin)
                torch.cuda.synchronize()
                self._hg = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self._hg, stream=s):
                    _, self._idx_out, _ = self.m.step(self._tin)
        self._pin_in.copy_(torch.from_numpy(idx_host[:, 0].astype(np.int64)))
        self._tin.copy_(self._pin_in, non_blocking=True)
        self._hg.replay()
        self._pin_out.copy_(self._idx_out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        idx_host[:] = self._pin_out.numpy().astype(np.uint32)

    def host_buffers(self, pinned):
        pass

    def io_bytes(self):
        return self.B * 8, self.B * self.k * 4

    def proxy_bytes(self):
        c = self.cfg
        return (c.layers * c.ffn * (c.d // 2 + 4) + c.vocab * (c.d // 2 + 4)) / (c.layers + 1)

    def step_bytes(self, x):
        return self.m.step_bytes(), 0, 0

    def recall(self, x):
        if self.world > 1:
            return None
        r = self.m.stage_recall(self.tok0)
        self.stage_rec = r
        return r["softmax"]

    def config(self):
        c = self.cfg
        return {"workload": "cfg5 decode step, 18-layer ReLU decoder (BASELINE.json configs[4])", "layers": c.layers,
                "d": c.d, "heads": c.heads, "ffn": c.ffn, "vocab": c.vocab, "kv_cache": c.ctx_len,
                "ffn_k": c.ffn_k, "ffn_k_prime": c.ffn_k_prime, "vocab_k": c.vocab_k,
                "vocab_k_prime": c.vocab_k_prime, "global_batch": self.B,
                "weights": "random-init bf16 (attention N(0,1/d); FFN cfg2 family; vocab cfg3 family, tied embedding)",
                "dense_parts": "RMSNorm, QKV/O projections (cuBLAS via torch), SDPA attention (library)",
                "recall_oracle": "same model with exact top-k FFN units and exact logits (teacher-forced per stage)",
                "stage_recall": getattr(self, "stage_rec", None),
                "l2": "working set ~3.2 GB + KV cache > 126 MB L2", "select": "exact top-k'"}


def make_workload(args, world=1, rank=0):
    B = B_default(args)
    if args.workload == "cfg3":
        return SoftmaxWorkload(B, select=args.select, world=world, rank=rank)
    if args.workload == "cfg1":
        return LowRankSoftmaxWorkload(B)
    if args.workload == "cfg4":
        return DaSoftmaxWorkload(B, world, rank)
    if args.workload == "cfg5":
        return DecoderWorkload(B, world, rank)
    return FfnWorkload(B)


def B_default(args):
    return args.batch or {"cfg2": 8, "cfg3": 32, "cfg1": 1, "cfg4": 16, "cfg5": 1}[args.workload]


# ------------------------------------------------------------- reference ---
def make_ref_runner(wl, host, threads):
    """The reference's own CPU implementation of the workload's path:
    oracle/_ref (the unmodified reference headers compiled behind a C shim)
    when it was built, else the C restatement (one thread). `host` holds the
    workload's weights as host arrays (made with plain torch, never through
    this repo's package); the int4 proxy is built by the reference's own
    quantize_int4 (approx.hpp:49-65). Returns (run(xb), threads, kind, desc);
    queries of one batch run on `threads` host threads (the reference API is
    pure and reentrant)."""
    import oracle as O
    kind = "reference" if O.ref_available() else "port"
    quant = O.ref_quantize_int4 if kind == "reference" else O.quantize_int4
    d = wl.d
    if wl.name == "cfg2":
        u, v = host["U"], host["V"]
        codes, scales = quant(u)
        desc = "hire::ffn_group_sparse (reference int4 scorer from hire::quantize_int4, fp32 x) on layer 0"
        if kind == "reference":
            rf = O.RefFFN(u, v, 1, 1)
            ra = O.RefScorer("quantized", codes=codes, scales=scales)

            def run(xb):
                out = np.empty((xb.shape[0], d), dtype=np.float32)
                O._ref_check(O.ref().ref_ffn_group_sparse_batch(
                    rf.h, ra.h, xb.ctypes.data_as(C.c_void_p), xb.shape[0], d, wl.k, wl.kp,
                    out.ctypes.data_as(C.c_void_p), threads))
            run._keep = (rf, ra)
        else:
            def run(xb):
                for b in range(xb.shape[0]):
                    O.ffn_group_sparse(u, v, xb[b], O.q4_scores_fpx(codes, scales, xb[b], 1), wl.k, wl.kp, 1, 1)
            threads = 1
        return run, threads, kind, desc
    W = host["W"]
    if wl.lowrank:
        z1, z2 = host["z1"], host["z2"]
        desc = "hire::hire_topk (reference low-rank scorer, exact top-k')"
    else:
        codes, scales = quant(W)
        desc = "hire::hire_topk (reference int4 scorer from hire::quantize_int4, fp32 x, exact top-k')"
    if kind == "reference":
        rm = O.RefMatrix(W)
        ra = (O.RefScorer("lowrank", z1=z1, z2=z2) if wl.lowrank else
              O.RefScorer("quantized", codes=codes, scales=scales))

        def run(xb):
            idx = np.empty((xb.shape[0], wl.k), dtype=np.uint32)
            val = np.empty((xb.shape[0], wl.k), dtype=np.float32)
            O._ref_check(O.ref().ref_hire_topk_batch(
                rm.h, ra.h, xb.ctypes.data_as(C.c_void_p), xb.shape[0], d, wl.k, wl.kp, 0,
                idx.ctypes.data_as(C.c_void_p), val.ctypes.data_as(C.c_void_p), threads))
        run._keep = (rm, ra)
    else:
        def run(xb):
            for b in range(xb.shape[0]):
                s = (O.lowrank_scores(z1, z2, xb[b], 0) if wl.lowrank else O.q4_scores_fpx(codes, scales, xb[b], 0))
                O.hire_topk(W, xb[b], s, wl.k, wl.kp, 0)
        threads = 1
    return run, threads, kind, desc


def host_queries(wl, n, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n, wl.d)) * wl.query_scale()).astype(np.float32)


def cpu_baseline(wl, host, seconds):
    """Bounded sample (~`seconds` of host work): batches of `threads` queries."""
    threads = os.cpu_count() or 1
    run, threads, kind, desc = make_ref_runner(wl, host, threads)
    xb = host_queries(wl, threads)
    t0 = time.perf_counter()
    run(xb)
    t1 = time.perf_counter() - t0
    reps = max(1, int(seconds / max(t1, 1e-6)))
    t0 = time.perf_counter()
    for _ in range(reps):
        run(xb)
    el = time.perf_counter() - t0
    n = reps * xb.shape[0]
    return n / el, threads, kind, f"{desc}: {n} queries in {el:.1f} s on {threads} host threads"


def measured_traffic(wl, batch):
    """DRAM bytes per launch of the roofline kernel from one committed
    `ncu --set full` capture (profiles/traffic.json), for the workload and
    batch it was captured at; None otherwise."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        return None
    e = t.get(f"{wl.name}_b{batch}") or (t.get(wl.name) if t.get(wl.name, {}).get("batch") == batch else None)
    return e["bytes"] if e else None


def pipelined_e2e(wl, H, device, xh, K, n_warm, pinned, lanes, serial):
    """The e2e metric with `lanes` host calls in flight: one host thread, one
    hire context (own stream, own workspaces and host-call graphs) and one set
    of pinned buffers per lane; lane l serves steps l, l + lanes, ... through
    the same blocking C-ABI call (ctypes drops the GIL inside it). Every step
    still fetches its own inputs from pinned host memory and writes its own
    results back inside the timed region; what changes is that one call's
    narrow tail (selector finisher, final top-k, result write-back, host
    wake-up) runs under the next call's proxy stream instead of on an idle
    GPU. Returns tokens/s and checks each lane's last result against the
    serial call on the same input."""
    import copy
    import threading
    lanes = min(lanes, K)  # every lane gets at least one step
    if lanes < 2:
        return None
    oa0, ob0, hctx0 = serial
    lw = []
    for l in range(lanes):
        w2 = copy.copy(wl)
        for a_ in ("_hp", "_hn", "_hr", "_hv", "_xd"):
            w2.__dict__.pop(a_, None)
        w2.host_buffers(pinned)
        lw.append((w2, H.Context(device, torch.cuda.Stream()), pinned(oa0.shape, torch.int32).view(np.uint32),
                   pinned(ob0.shape, torch.float32)))

    def lane(l, first, n, gate=None):
        w2, ctx, oa, ob = lw[l]
        if gate is not None:
            gate.wait()
        for i in range(first + l, first + n, lanes):
            w2.host_step(i, xh[i % len(xh)], oa, ob, ctx)

    for l in range(lanes):  # one lane at a time first: lazily built workspaces and graphs
        lane(l, 0, lanes * n_warm)
    n = K - K % lanes
    for timed in (False, True):
        gate = threading.Barrier(lanes + 1)
        th = [threading.Thread(target=lane, args=(l, lanes * n_warm, n, gate)) for l in range(lanes)]
        for t in th:
            t.start()
        gate.wait()
        t0 = time.perf_counter()
        for t in th:
            t.join()
        dt = time.perf_counter() - t0
    ok = True
    for l in range(lanes):  # lane l's last step, again through the serial context
        i = lanes * n_warm + n - lanes + l
        wl.host_step(i, xh[i % len(xh)], oa0, ob0, hctx0)
        ok = ok and np.array_equal(oa0, lw[l][2]) and np.array_equal(ob0.view(np.uint32), lw[l][3].view(np.uint32))
    return {"value": round(wl.B * n / dt, 2), "in_flight": lanes, "steps": n,
            "equals_serial_call": bool(ok)}


# ------------------------------------------------------------------- ours ---
def run_ours(args):
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2402_09360_b200 as H
    H.lib()
    wl = make_workload(args, world, rank)
    wl.attach(H)
    K, W = args.steps, args.warmup
    xs = wl.inputs(K + W)
    # Each timed step replays from one CUDA graph holding the K calls
    # (graphs instead of a tracing compiler: no host work between kernels).
    # Warm-up runs eagerly on the capture stream first, so every workspace
    # exists before capture.
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        ctx = H.default_context()
        for i in range(W):
            wl.step(i, xs[i])
    torch.cuda.synchronize()
    n0 = ctx.launches()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=cs):
        for i in range(K):
            out_single = wl.step(W + i, xs[W + i])
    launches = ctx.launches() - n0
    for _ in range(2):
        graph.replay()  # graph warm-up
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t_end = time.perf_counter() + 1.0
        while time.perf_counter() < t_end:  # soak: steady clocks before timing
            graph.replay()
            torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    ms_step = ms / K
    # tokens the whole job decoded: strong scaling (DA over one batch) counts
    # the batch once; weak scaling (independent replicas) counts every rank's
    tokens = wl.B * K * (1 if wl.scaling == "strong" else world)
    value = tokens / (ms / 1e3)
    single = {"ms_per_step": round(ms_step, 5), "value": round(value, 2)}
    S = min(args.streams, K) if (world == 1 and not getattr(wl, "da", False) and wl.name != "cfg5") else 1
    if S > 1:
        # The same K steps dealt over S streams (one hire context and workspace
        # set per stream) inside one graph: independent batches, so one
        # batch's narrow tail (finisher, final top-k: a few dozen CTAs) runs
        # under another batch's proxy / gather stream instead of on an idle GPU.
        try:
            sides = [torch.cuda.Stream() for _ in range(S - 1)]
            for st in sides:
                st.wait_stream(cs)
                with torch.cuda.stream(st):
                    H.default_context()
                    for i in range(max(W, 2)):
                        wl.step(i, xs[i])
            torch.cuda.synchronize()
            mgraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(mgraph, stream=cs):
                for st in sides:
                    st.wait_stream(cs)
                for l, st in enumerate([cs] + sides):
                    with torch.cuda.stream(st):
                        for i in range(l, K, S):
                            o_ = wl.step(W + i, xs[W + i])
                            if i == K - 1:
                                out_multi = o_
                for st in sides:
                    cs.wait_stream(st)
            for _ in range(3):
                mgraph.replay()
            torch.cuda.synchronize()
            t_end = time.perf_counter() + 0.5
            while time.perf_counter() < t_end:
                mgraph.replay()
                torch.cuda.synchronize()
            e0.record()
            mgraph.replay()
            e1.record()
            torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
            flat = lambda o: [t for t in (o if isinstance(o, (tuple, list)) else [o]) if torch.is_tensor(t)]  # noqa: E731
            streams_equal = all(torch.equal(a_, b_) for a_, b_ in zip(flat(out_single), flat(out_multi)))
            if not streams_equal:
                raise RuntimeError("multi-stream step result differs from the single-stream one")
            ms = e0.elapsed_time(e1)
            ms_step = ms / K
            value = tokens / (ms / 1e3)
        except Exception as e:  # the single-stream number stands
            print(f"[bench] multi-stream graph failed ({e}); single stream", file=sys.stderr)
            S = 1

    # stage times: the same K steps captured with CUDA events bracketing
    # every stage (event-record nodes inside the graph), replayed once
    prof = None
    try:
        with torch.cuda.stream(cs):
            ctx.profile_read()
            ctx.set_profiling(True)
        pgraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(pgraph, stream=cs):
            for i in range(K):
                wl.step(W + i, xs[W + i])
        with torch.cuda.stream(cs):
            ctx.set_profiling(False)
        pgraph.replay()
        torch.cuda.synchronize()
        prof = ctx.profile_read()
        prof["_graph"] = (1.0, 1)
    except Exception as e:  # fall back to eager profiling
        print(f"[bench] graph stage profiling failed ({e}); eager", file=sys.stderr)
        prof = None
    if not prof or "proxy" not in prof:
        with torch.cuda.stream(cs):
            ctx.set_profiling(True)
            ctx.profile_read()
            for i in range(K):
                wl.step(W + i, xs[W + i])
            ctx.set_profiling(False)
            prof = ctx.profile_read()
    stage_us = {k: v[0] * 1e3 / K for k, v in prof.items() if not k.startswith("_")}

    # device timeline of one step (%globaltimer, first CTA start -> last CTA
    # end per kernel; hire_debug_ktrace) replayed from a one-step graph
    spans = None
    try:
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1, stream=cs):
            wl.step(W, xs[W])
        best = None
        for _ in range(3):
            for _ in range(2):
                g1.replay()
            torch.cuda.synchronize()
            ctx.ktrace(1)
            g1.replay()
            torch.cuda.synchronize()
            sp = ctx.ktrace(2)
            ctx.ktrace(0)
            kk = "lr_score" if wl.lowrank else "proxy"
            if kk in sp and (best is None or sp[kk][1] - sp[kk][0] < best[kk][1] - best[kk][0]):
                best = sp
        spans = best
    except Exception as e:
        print(f"[bench] device timeline failed ({e})", file=sys.stderr)

    peaks = load_peaks()
    step_b, nu, nv = wl.step_bytes(xs[W])
    kbytes = wl.kernel_bytes(nu) if hasattr(wl, "kernel_bytes") else {}
    if getattr(wl, "roof_stage", None) in prof:
        # the workload's dominant kernel is not the proxy (cfg4: the gather
        # recompute is ~3/4 of the step in the ncu launch list)
        kname, kkey = wl.roof_kernel, wl.roof_stage
        pb = kbytes[wl.roof_stage]
    else:
        kname, kkey = wl.proxy_kernel, ("lr_score" if wl.lowrank else "proxy")
        pb = wl.proxy_bytes()
    k_us = prof["proxy" if kkey in ("proxy", "lr_score") else kkey][0] * 1e3 / \
        max(prof["proxy" if kkey in ("proxy", "lr_score") else kkey][1], 1)
    achieved = pb / (k_us * 1e-6) / 1e9
    dspan = None
    if spans and kkey in spans and getattr(wl, "span_kernel", "x") is not None:
        dspan = spans[kkey][1] - spans[kkey][0]
    rec = wl.recall(xs[W])

    # end-to-end through the C ABI with host buffers (copies inside)
    hctx = H.Context(local)
    bi, bo = wl.io_bytes()

    def pinned(shape, dt):
        return torch.empty(shape, dtype=dt).pin_memory().numpy()
    xh = []
    for i in range(min(K, 64)):
        if xs[W + i] is None:
            xh.append(None)
            continue
        a_ = pinned(tuple(xs[W + i].shape), torch.float32)
        a_[:] = xs[W + i].cpu().numpy()
        xh.append(a_)
    oa = pinned((wl.B, wl.k), torch.int32).view(np.uint32)
    ob = pinned((wl.B, wl.d) if wl.name == "cfg2" else (wl.B, wl.k), torch.float32)
    wl.host_buffers(pinned)
    n_cycle = len(getattr(wl, "layers", None) or getattr(wl, "copies", None) or [0])
    n_warm = max(W, 2 * n_cycle + 1)
    if wl.name == "cfg5":  # the decode chain's tokens travel in oa[:, 0]
        oa[:, 0] = wl.tok0.cpu().numpy().astype(np.uint32)
    for i in range(n_warm):
        wl.host_step(i, xh[i % len(xh)], oa, ob, hctx)
    barrier(world)
    t0 = time.perf_counter()
    for i in range(K):
        wl.host_step(n_warm + i, xh[i % len(xh)], oa, ob, hctx)
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    e2e = wl.B * K * (1 if wl.scaling == "strong" else world) / e2e_s
    pipe = None
    if world == 1 and not getattr(wl, "da", False) and wl.name != "cfg5" and args.in_flight > 1:
        try:
            pipe = pipelined_e2e(wl, H, local, xh, K, n_warm, pinned, args.in_flight, (oa, ob, hctx))
        except Exception as e:  # the serial number stands
            print(f"[bench] pipelined e2e failed ({e})", file=sys.stderr)

    par = ("single GPU" + (" (HIRE_BENCH_DA=1: da_topk with a 1-rank NCCL communicator — validation run)"
                           if getattr(wl, "da", False) else "")) if world == 1 else (
        f"DA-TOP-k over {world} GPUs (rows sharded, ncclAllGather of keys)" if wl.scaling == "strong"
        else f"replicas x{world}")
    uniq = nu if not isinstance(nu, tuple) else {"u_rows": nu[0], "v_rows": nu[1]}
    line = {
        "metric": METRIC,
        "value": round(value, 2), "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": round(ms_step, 5), "us_per_token": round(ms_step * 1e3 / wl.B, 4),
        "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None, "dtype": wl.dtype,
        "data": "synthetic (seeded random-init weights of the BASELINE family; random queries)",
        "config": {**wl.config(), "parallelism": par},
        "recall_at_k": round(rec, 5) if rec is not None else None,
        "roofline": {"bound": "hbm", "kernel": kname,
                     "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": measured_traffic(wl, wl.B),
                     "bytes_per_launch": pb, "avg_launch_us": round(k_us, 3),
                     "timing": "CUDA events around the kernel's stage inside the replayed graph (includes its launch "
                               "latency: the event nodes break the programmatic-dependent-launch overlap)",
                     "device_span_us": round(dspan, 3) if dspan else None,
                     "frac_device_span": round(pb / (dspan * 1e-6) / 1e9 / peaks["hbm_gbs"], 4) if dspan else None,
                     "peak_src": peaks["src"]},
        "step_timeline_us": {k: v for k, v in (spans or {}).items() if isinstance(v, tuple)},
        "kernel_roofline": {k: {"bytes": b, "bytes_model": "unique rows of the batch x row bytes",
                                "span_us": round(spans[k][1] - spans[k][0], 3),
                                "gbs": round(b / ((spans[k][1] - spans[k][0]) * 1e-6) / 1e9, 1),
                                "frac": round(b / ((spans[k][1] - spans[k][0]) * 1e-6) / 1e9 / peaks["hbm_gbs"], 4)}
                            for k, b in kbytes.items() if spans and k in spans and spans[k][1] > spans[k][0]},
        "step_roofline": {"bytes": step_b, "unique_rows": uniq,
                          "model": "roofline_bytes: proxy incl. scales + unique gathered rows (+ all-gather)",
                          "achieved_gbs": round(step_b / (ms_step * 1e-3) / 1e9, 1),
                          "frac": round(step_b / (ms_step * 1e-3) / 1e9 / peaks["hbm_gbs"], 4)},
        "streams": S,
        "streams_note": ("the K timed steps are dealt over %d streams inside one CUDA graph (one hire context and "
                         "workspace set per stream; independent batches, every step does the full work and the last "
                         "step's result is checked equal to the single-stream graph's): tails of one batch overlap the "
                         "HBM-bound kernels of another. value/ms_per_step/step_roofline are throughput over the K steps; "
                         "single_stream is one batch at a time" % S) if S > 1 else "one batch at a time",
        "single_stream": single,
        "stage_us_per_step": {k: round(v, 3) for k, v in stage_us.items()},
        "stage_timing": "CUDA events inside the replayed graph" if "_graph" in prof else "CUDA events, eager launches",
        "e2e": {"value": pipe["value"] if pipe else round(e2e, 2), "unit": "tokens/s", "h2d_bytes_per_step": bi,
                "d2h_bytes_per_step": bo,
                "in_flight": pipe["in_flight"] if pipe else 1,
                "single_call": {"value": round(e2e, 2), "us_per_call": round(e2e_s / K * 1e6, 2),
                                "note": "one blocking host call at a time (the latency view)"},
                "mode": ("%d blocking host calls in flight: one host thread + one hire context (own stream, "
                         "workspaces, call graph, pinned buffers) per lane; every step fetches its own inputs "
                         "and writes its own results inside the timed region" % pipe["in_flight"])
                        if pipe else "one blocking host call at a time",
                "path": "C-ABI host call (hire_topk_host / hire_ffn_host) with pinned host buffers"
                        if not getattr(wl, "da", world > 1) else "python parallel.da_topk with pinned copies",
                "pipelined": pipe},
        "gpu_launches": int(launches),
        "select_fallbacks": int(ctx.select_fallbacks()),  # queries that took the slow exact path (whole run)
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and wl.name != "cfg5":
        v, cores, kind, desc = cpu_baseline(wl, wl.ref_host(), args.cpu_seconds)
        line["cpu_baseline"] = {"value": round(v, 3), "unit": "tokens/s", "cores": cores, "kind": kind,
                                "sample": desc}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# -------------------------------------------------------------- reference ---
def run_reference(args):
    """--impl reference: the reference's CPU implementation of the same
    workload (oracle/_ref: the unmodified reference headers) on all host
    threads. Weights come from the same torch generators as our arm, copied
    to the host; the int4 proxy is built by the reference's quantize_int4.
    This arm never imports paper_2402_09360_b200 (nor loads its .so). Each
    step = one batch of max(B, threads) queries. Rank 0 only."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    if args.workload == "cfg5":
        print(json.dumps({"impl": "reference", "unavailable": "the reference has no decoder (cfg5 glue is not in "
                                                              "the reference library)"}), flush=True)
        return
    torch.cuda.set_device(local)
    wl = make_workload(args)  # plain torch tensors; no attach()
    host = wl.ref_host()
    wl.__dict__.pop("Wt", None)  # the device copy is no longer needed
    torch.cuda.empty_cache()
    threads = os.cpu_count() or 1
    run, threads, kind, desc = make_ref_runner(wl, host, threads)
    nq = max(wl.B, threads)
    K, W = args.steps, args.warmup
    xs = host_queries(wl, (K + W) * nq, seed=1).reshape(K + W, nq, wl.d)
    for i in range(W):
        run(xs[i])
    t0 = time.perf_counter()
    for i in range(K):
        run(xs[W + i])
    el = time.perf_counter() - t0
    v = nq * K / el
    line = {"impl": "reference", "metric": METRIC,
            "value": round(v, 3), "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": round(el * 1e3 / K, 3), "higher_is_better": True, "scaling": wl.scaling,
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic (same torch generators as our arm)",
            "config": {**wl.config(), "parallelism": f"{threads} host threads", "queries_per_step": nq,
                       "reference_proxy": "reference scorer with fp32 x (approx.hpp:395-403); ours scores int8 x"},
            "cpu_baseline": {"value": round(v, 3), "unit": "tokens/s", "cores": threads, "kind": kind,
                             "sample": f"{desc}: {K} steps x {nq} queries"},
            "e2e": {"value": round(v, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--select", default="exact", choices=["exact", "bucketed"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=6,
                    help="streams the K timed steps are dealt over inside the graph (independent batches)")
    ap.add_argument("--in-flight", type=int, default=6,
                    help="host calls in flight for the e2e number (1: one blocking call at a time)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
