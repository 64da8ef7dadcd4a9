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
