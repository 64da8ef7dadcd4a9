"""Decoder glue for BASELINE.json configs[4] (SURVEY.md §8 f, rank 3): one
greedy decode step of a ReLU decoder whose FFNs are HiRE-FFN layers and
whose output layer is HiRE-softmax. Not in the reference (no parity there):
the dense parts — RMSNorm, the QKV / output projections (cuBLAS through
torch.matmul) and attention over a KV cache (torch SDPA / flash) — are
library code; every HiRE stage runs in libhire_cuda.so. The dense oracle is
the same model with k = k' = all units / all vocab rows
(tests/test_decoder.py).

DA-TOP-k sharding (BASELINE configs[4]: FFN hidden units and vocabulary
sharded D ways): with a communicator (`comm`, one process per GPU) every FFN
layer runs `parallel.da_group_sparse` over this rank's hidden-unit shard
(local quotas, one grouped all-gather of unit ids + partial outputs, rank-
order sum: every rank ends with the same residual stream) and the output
layer `parallel.da_topk` over this rank's vocabulary shard (global merge).
`emulate=D` runs the same D-shard algorithm on one GPU
(`da_group_sparse_emulated` / `da_topk_emulated`) for tests. Attention and
the tied embedding are replicated."""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import torch
import torch.nn.functional as F

from . import _lib as L
from .api import (ApproxScorer, GroupedFFN, HireConfig, ScoreMatrix, da_group_sparse_emulated, da_topk_emulated,
                  ffn_group_sparse, hire_topk)


@dataclass
class DecoderConfig:
    layers: int = 18
    d: int = 2048
    heads: int = 16
    ffn: int = 8192
    vocab: int = 256000
    ctx_len: int = 1024
    ffn_k: int = 410        # top-5% of 8192 (exact)
    ffn_k_prime: int = 820  # 10% candidates from the int4 proxy
    vocab_k: int = 64
    vocab_k_prime: int = 1024


@dataclass
class _Layer:
    wqkv: torch.Tensor      # [3d, d] bf16
    wo: torch.Tensor        # [d, d] bf16
    ffn: GroupedFFN
    proxy: ApproxScorer
    k_cache: torch.Tensor   # [B, H, T, hd] bf16
    v_cache: torch.Tensor
    ffn_shard: Optional[GroupedFFN] = None     # this rank's hidden units (comm mode)
    proxy_shard: Optional[ApproxScorer] = None


def _rmsnorm(h: torch.Tensor) -> torch.Tensor:
    hf = h.float()
    return hf * torch.rsqrt(hf.pow(2).mean(-1, keepdim=True) + 1e-6)


class HireDecoder:
    """Random-init weights (seeded): attention N(0, 1/d); FFN U, V the cfg2
    family (N(0, 1/d) + 3x rank-128); vocab rows the cfg3 family (rank-256 +
    0.1 N(0, 1)), tied with the token embedding; KV caches N(0, 1)."""

    def __init__(self, cfg: DecoderConfig, batch: int, seed: int = 0, dtype=torch.bfloat16, comm=None,
                 emulate: int = 1):
        self.cfg, self.B = cfg, batch
        self.comm, self.emulate = comm, emulate
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        d, hd = cfg.d, cfg.d // cfg.heads
        g = torch.Generator(device="cuda").manual_seed(seed)

        def randn(*shape, scale=1.0):
            return (torch.randn(*shape, device="cuda", generator=g) * scale).to(dtype).contiguous()

        self.layers: List[_Layer] = []
        r = min(128, cfg.ffn, d)
        for _ in range(cfg.layers):
            def ffn_mat():
                base = torch.randn(cfg.ffn, d, device="cuda", generator=g) / d ** 0.5
                A = torch.randn(cfg.ffn, r, device="cuda", generator=g)
                Bm = torch.randn(r, d, device="cuda", generator=g)
                return (base + 3.0 * (A @ Bm) / (r * d) ** 0.5).to(dtype).contiguous()
            f = GroupedFFN(ScoreMatrix(ffn_mat()), ScoreMatrix(ffn_mat()), 1, "relu")
            self.layers.append(_Layer(randn(3 * d, d, scale=d ** -0.5), randn(d, d, scale=d ** -0.5), f,
                                      ApproxScorer.quantize(f.u),
                                      randn(batch, cfg.heads, cfg.ctx_len, hd), randn(batch, cfg.heads, cfg.ctx_len, hd)))
        rv = min(256, cfg.vocab, d)
        W = torch.empty(cfg.vocab, d, device="cuda", dtype=dtype)
        Bv = torch.randn(rv, d, device="cuda", generator=g)
        for s in range(0, cfg.vocab, 32768):
            e = min(cfg.vocab, s + 32768)
            A = torch.randn(e - s, rv, device="cuda", generator=g)
            W[s:e] = (A @ Bv / rv ** 0.5 + 0.1 * torch.randn(e - s, d, device="cuda", generator=g)).to(dtype)
        self.vocab = ScoreMatrix(W)
        self.vocab_proxy = ApproxScorer.quantize(self.vocab)
        self.embed = W  # tied
        self.softmax_cfg = HireConfig(k=cfg.vocab_k, k_prime=cfg.vocab_k_prime, x_mode=L.X_INT8)
        if comm is not None:
            # this rank's shards (width rule, distributed.hpp:53-57): row
            # views of the replicated weights, each with its own int4 proxy
            from .parallel import shard_range
            for lay in self.layers:
                f0, w0 = shard_range(cfg.ffn, self.world, self.rank)
                lay.ffn_shard = GroupedFFN(lay.ffn.u.slice_cols(f0, w0), lay.ffn.v.slice_cols(f0, w0), 1, "relu")
                lay.proxy_shard = ApproxScorer.quantize(lay.ffn_shard.u)
            v0, vw = shard_range(cfg.vocab, self.world, self.rank)
            self.vocab_shard = self.vocab.slice_cols(v0, vw)
            self.vocab_proxy_shard = ApproxScorer.quantize(self.vocab_shard)

    def attention(self, lay: _Layer, a: torch.Tensor) -> torch.Tensor:
        """Dense attention for the new token over the KV cache (the newest
        key/value overwrite the last cache slot: a fixed-length decode window)."""
        cfg = self.cfg
        hd = cfg.d // cfg.heads
        qkv = a.to(lay.wqkv.dtype) @ lay.wqkv.t()
        q, k, v = qkv.view(self.B, 3, cfg.heads, hd).unbind(1)
        lay.k_cache[:, :, -1] = k
        lay.v_cache[:, :, -1] = v
        o = F.scaled_dot_product_attention(q.unsqueeze(2), lay.k_cache, lay.v_cache)
        return o.reshape(self.B, cfg.d) @ lay.wo.t()

    def step(self, tokens: torch.Tensor, ffn_k: Optional[int] = None, ffn_k_prime: Optional[int] = None,
             softmax_cfg: Optional[HireConfig] = None):
        """One greedy decode step for B tokens -> (next tokens [B], top-k
        indices [B, k], top-k logits [B, k])."""
        cfg = self.cfg
        kk = ffn_k or cfg.ffn_k
        kp = ffn_k_prime or cfg.ffn_k_prime
        sm = softmax_cfg or self.softmax_cfg
        h = self.embed[tokens].float()
        for lay in self.layers:
            h = h + self.attention(lay, _rmsnorm(h)).float()
            h = h + self._ffn(lay, _rmsnorm(h).contiguous(), kk, kp)
        z = _rmsnorm(h).contiguous()
        if self.comm is not None:
            from .parallel import da_topk
            ti, tv, _ = da_topk(self.vocab_shard, self.vocab_proxy_shard, self.cfg.vocab, z, sm, self.comm,
                                merge=L.MERGE_GLOBAL)
            return ti[:, 0], ti, tv
        if self.emulate > 1:
            ti, tv, _ = da_topk_emulated(self.vocab, self.vocab_proxy, z, self.emulate, sm, merge=L.MERGE_GLOBAL,
                                         uneven=True)
            return ti[:, 0], ti, tv
        r = hire_topk(z, self.vocab, self.vocab_proxy, sm, want_candidates=False)
        return r.top_idx[:, 0], r.top_idx, r.top_val

    def _ffn(self, lay: _Layer, x: torch.Tensor, k: int, kp: int) -> torch.Tensor:
        """HiRE-FFN of one layer: whole (one GPU), DA-sharded across ranks
        (da_group_sparse, distributed.hpp:145-206), or its D-shard emulation."""
        if self.comm is not None:
            from .parallel import da_group_sparse
            out, _ = da_group_sparse(lay.ffn_shard, lay.proxy_shard, self.cfg.ffn, x, k, kp, self.comm,
                                     x_mode=L.X_INT8, uneven=True)
            return out
        if self.emulate > 1:
            out, _ = da_group_sparse_emulated(lay.ffn, x, lay.proxy, k, kp, self.emulate, x_mode=L.X_INT8, uneven=True)
            return out
        out, _ = ffn_group_sparse(lay.ffn, x, lay.proxy, k, kp, x_mode=L.X_INT8)
        return out

    def dense_step(self, tokens: torch.Tensor, ffn_k: Optional[int] = None):
        """The dense oracle (fp32 torch arithmetic on the same weights): every
        FFN unit, or with ffn_k the exact top-k units per token (ffn_topk,
        ffn.hpp:78-100 — what HiRE-FFN approximates); exact logits over the
        whole vocab."""
        h = self.embed[tokens].float()
        for lay in self.layers:
            h = h + self.attention(lay, _rmsnorm(h)).float()
            x = _rmsnorm(h)
            act = torch.relu(x @ lay.ffn.u.tensor.float().t())
            if ffn_k is not None:
                thr = torch.topk(act, ffn_k, dim=-1).values[:, -1:]
                act = torch.where(act >= thr, act, torch.zeros_like(act))
            h = h + act @ lay.ffn.v.tensor.float()
        logits = _rmsnorm(h) @ self.vocab.tensor.float().t()
        val, idx = torch.topk(logits, self.cfg.vocab_k, dim=-1)
        return idx[:, 0], idx, val

    def stage_recall(self, tokens: torch.Tensor) -> dict:
        """Teacher-forced recall of every HiRE stage on the exact-top-k model's
        own hidden states: per layer, |HiRE-FFN units ∩ exact top-k units| / k;
        at the output, |HiRE-softmax top-k ∩ exact top-k| / k. (With random
        weights the two residual streams themselves decorrelate over 18
        layers, so end-to-end token agreement says nothing about the stages.)"""
        cfg = self.cfg
        h = self.embed[tokens].float()
        ffn_rec = []
        for lay in self.layers:
            h = h + self.attention(lay, _rmsnorm(h)).float()
            x = _rmsnorm(h).contiguous()
            _, sel = ffn_group_sparse(lay.ffn, x, lay.proxy, cfg.ffn_k, cfg.ffn_k_prime, x_mode=L.X_INT8)
            act = torch.relu(x @ lay.ffn.u.tensor.float().t())
            top = torch.topk(act, cfg.ffn_k, dim=-1).indices
            ffn_rec.append(sum(len(set(sel[b].tolist()) & set(top[b].tolist())) for b in range(self.B)) /
                           (self.B * cfg.ffn_k))
            thr = torch.topk(act, cfg.ffn_k, dim=-1).values[:, -1:]
            h = h + torch.where(act >= thr, act, torch.zeros_like(act)) @ lay.ffn.v.tensor.float()
        z = _rmsnorm(h).contiguous()
        r = hire_topk(z, self.vocab, self.vocab_proxy, self.softmax_cfg, want_candidates=False)
        ex = torch.topk(z @ self.vocab.tensor.float().t(), cfg.vocab_k, dim=-1).indices
        sm = sum(len(set(r.top_idx[b].tolist()) & set(ex[b].tolist())) for b in range(self.B)) / (self.B * cfg.vocab_k)
        return {"ffn_layers_mean": float(sum(ffn_rec) / len(ffn_rec)), "ffn_layers_min": float(min(ffn_rec)),
                "softmax": float(sm)}

    def step_bytes(self) -> int:
        """Roofline bytes of one step (SURVEY.md §8 d): attention weights + KV
        cache + HiRE-FFN (proxy + k' U rows + k V rows per token) per layer,
        + the vocab proxy and k' gathered vocab rows per token."""
        cfg = self.cfg
        d, es = cfg.d, 2
        proxy_ffn = cfg.ffn * (d // 2 + 4)
        per_layer = (4 * d * d * es + 2 * self.B * cfg.ctx_len * d * es + proxy_ffn +
                     self.B * (cfg.ffn_k_prime + cfg.ffn_k) * d * es)
        return cfg.layers * per_layer + cfg.vocab * (d // 2 + 4) + self.B * cfg.vocab_k_prime * d * es
