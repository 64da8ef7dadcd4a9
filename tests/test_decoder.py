"""Decoder glue (BASELINE configs[4], SURVEY.md §8 f rank 3) against its
dense oracle: the same model with every FFN unit and exact logits over the
whole vocabulary. With k = k' = all units and k' = V the HiRE step must pick
the dense step's tokens (the HiRE stages then compute exactly the dense
sums, up to fp32 summation order); at the production quotas the final
top-k must match the exact-top-k model's (ffn_topk FFNs, exact logits)
with high recall."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _small():
    from paper_2402_09360_b200.decoder import DecoderConfig
    return DecoderConfig(layers=2, d=256, heads=4, ffn=1024, vocab=8192, ctx_len=64, ffn_k=51, ffn_k_prime=102,
                         vocab_k=16, vocab_k_prime=256)


def test_decoder_full_quotas_equal_dense(H):
    from paper_2402_09360_b200.decoder import HireDecoder
    cfg = _small()
    m = HireDecoder(cfg, batch=4, seed=1, dtype=torch.float32)
    tok = torch.randint(0, cfg.vocab, (4,), device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    full = H.HireConfig(k=cfg.vocab_k, k_prime=cfg.vocab, x_mode=H.X_INT8)
    nxt, idx, val = m.step(tok, ffn_k=cfg.ffn, ffn_k_prime=cfg.ffn, softmax_cfg=full)
    dn, didx, dval = m.dense_step(tok)
    assert torch.equal(nxt, dn.to(nxt.dtype))
    torch.testing.assert_close(val, dval, rtol=1e-4, atol=1e-4)


def test_decoder_production_quotas(H):
    from paper_2402_09360_b200.decoder import HireDecoder
    cfg = _small()
    m = HireDecoder(cfg, batch=16, seed=3)
    tok = torch.randint(0, cfg.vocab, (16,), device="cuda", generator=torch.Generator(device="cuda").manual_seed(4))
    nxt, idx, val = m.step(tok)
    dn, didx, _ = m.dense_step(tok, ffn_k=cfg.ffn_k)
    assert idx.shape == (16, cfg.vocab_k)
    # recall@k of the final top-k against the exact-top-k model (what the
    # HiRE stages approximate: int4 proxy candidates, then exact top-k)
    rec = sum(len(set(idx[b].tolist()) & set(didx[b].tolist())) for b in range(16)) / (16 * cfg.vocab_k)
    assert rec > 0.8, rec


def test_decoder_sharded_one_rank_comm_equals_unsharded(H):
    """DA-sharded decoder step (da_group_sparse per FFN layer, da_topk over
    the vocabulary) through a 1-rank NCCL communicator — the full local ->
    all-gather -> merge chain of every stage — gives the unsharded step."""
    from paper_2402_09360_b200 import parallel as P
    from paper_2402_09360_b200.decoder import HireDecoder
    cfg = _small()
    comm = P.Communicator(1, 0)
    m0 = HireDecoder(cfg, batch=8, seed=5)
    m1 = HireDecoder(cfg, batch=8, seed=5, comm=comm)
    tok = torch.randint(0, cfg.vocab, (8,), device="cuda", generator=torch.Generator(device="cuda").manual_seed(6))
    for _ in range(2):
        n0, i0, v0 = m0.step(tok)
        n1, i1, v1 = m1.step(tok)
        assert torch.equal(i0.long(), i1.long()) and torch.equal(v0, v1)
        tok = n0.long()


@pytest.mark.parametrize("shards", [2, 4])
def test_decoder_emulated_shard_stages(H, shards):
    """The D-shard stages the sharded decoder runs (local quotas, uneven for
    k = 51; global merge for the vocabulary), teacher-forced on one hidden
    state: DA-FFN units and DA-softmax tokens against the exact top-k, and
    the emulated step runs end to end. (Per-shard quotas approximate the
    global top-k — distributed.hpp:172-201 — so a free-running sharded
    decode drifts from the unsharded one over layers.)"""
    from paper_2402_09360_b200.decoder import HireDecoder, _rmsnorm
    cfg = _small()
    m = HireDecoder(cfg, batch=16, seed=3, emulate=shards)
    g = torch.Generator(device="cuda").manual_seed(4)
    x = _rmsnorm(torch.randn(16, cfg.d, device="cuda", generator=g)).contiguous()
    lay = m.layers[0]
    _, sel = H.da_group_sparse_emulated(lay.ffn, x, lay.proxy, cfg.ffn_k, cfg.ffn_k_prime, shards, x_mode=H.X_INT8,
                                        uneven=True)
    act = torch.relu(x @ lay.ffn.u.tensor.float().t())
    top = torch.topk(act, cfg.ffn_k, dim=-1).indices
    rec = sum(len(set(sel[b].tolist()) & set(top[b].tolist())) for b in range(16)) / (16 * cfg.ffn_k)
    assert rec > 0.8, rec
    ti, tv, _ = H.da_topk_emulated(m.vocab, m.vocab_proxy, x, shards, m.softmax_cfg, merge=H.MERGE_GLOBAL)
    ex = torch.topk(x @ m.vocab.tensor.float().t(), cfg.vocab_k, dim=-1).indices
    rec_s = sum(len(set(ti[b].tolist()) & set(ex[b].tolist())) for b in range(16)) / (16 * cfg.vocab_k)
    assert rec_s > 0.9, rec_s
    tok = torch.randint(0, cfg.vocab, (16,), device="cuda", generator=g)
    nxt, idx, val = m.step(tok)
    assert idx.shape == (16, cfg.vocab_k) and bool(torch.all(val[:, :-1] >= val[:, 1:]))


@pytest.mark.parametrize("B", [1, 64])
def test_decoder_cfg5_full_size_stage_recall(H, B):
    """BASELINE configs[4] at its own shape (18 layers, d=2048, FFN 8192 at
    top-5% from 10% int4-proxy candidates, 16 heads x 1024-token KV cache,
    V=256000 HiRE-softmax k'=1024, k=64): every stage, teacher-forced on the
    exact-top-k model's hidden states, recovers the exact top-k units /
    tokens (recall of the FFN units and of the softmax top-k)."""
    from paper_2402_09360_b200.decoder import DecoderConfig, HireDecoder
    m = HireDecoder(DecoderConfig(), batch=B, seed=7)
    tok = torch.randint(0, 256000, (B,), device="cuda", generator=torch.Generator(device="cuda").manual_seed(8))
    r = m.stage_recall(tok)
    assert r["ffn_layers_mean"] > 0.98 and r["ffn_layers_min"] > 0.95, r
    assert r["softmax"] > 0.95, r
    nxt, idx, val = m.step(tok)
    assert idx.shape == (B, 64) and bool(torch.all(val[:, :-1] >= val[:, 1:]))
