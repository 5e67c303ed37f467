"""Llama decode E2E on cuda:0: the MACKO-linear model against the same model
with dense cuBLAS linears over identical weights, teacher-forced, at a reduced size; plus the
greedy-generation plumbing (device-side position / token, CUDA-graph replay)."""
import numpy as np
import pytest
import torch

from paper_2511_13061_b200 import llama as L

pytestmark = pytest.mark.gpu

SMALL = L.LlamaConfig(vocab=1000, hidden=512, layers=3, heads=4, inter=1376, max_len=32)  # head_dim 128


def _forced_logits(dec, tokens):
    out = []
    dec.reset()
    for t, tok in enumerate(tokens):
        dec.pos.fill_(t)
        dec.token.fill_(tok)
        dec.step(sample=False)
        out.append(dec.logits.float().clone())
    torch.cuda.synchronize()
    return torch.stack(out)


def test_macko_model_matches_dense_model(cuda):
    w = L.LlamaWeights(SMALL, density=0.5, device=cuda)
    tokens = [1, 17, 999, 3, 256, 42, 7, 500]
    ld = _forced_logits(L.LlamaDecoder(w, "dense"), tokens)
    lm = _forced_logits(L.LlamaDecoder(w, "macko"), tokens)
    assert torch.isfinite(lm).all() and torch.isfinite(ld).all()
    # same lossless weights; the models differ only by the fp32 summation order of each linear
    # (each within |dy| <= ulp16 + 2 n 2^-24 sum|a x|), compounded through 3 layers
    err = (lm - ld).abs().max().item()
    scale = ld.abs().max().item()
    assert err <= 2e-2 * scale, (err, scale)
    cos = torch.nn.functional.cosine_similarity(lm, ld, dim=1)
    assert (cos > 0.9999).all(), cos
    assert (lm.argmax(1) == ld.argmax(1)).float().mean() >= 0.75
    w.close()


def test_greedy_generation_graph(cuda):
    w = L.LlamaWeights(SMALL, density=0.5, device=cuda)
    dec = L.LlamaDecoder(w, "macko")
    secs = dec.generate(12)
    hist = dec.history[:12].cpu().numpy()
    assert secs > 0 and int(dec.pos.item()) == 12
    assert ((hist >= 0) & (hist < SMALL.vocab)).all()
    # stream launches without the graph reproduce the graph's tokens exactly
    dec2 = L.LlamaDecoder(w, "macko")
    dec2.reset()
    for _ in range(12):
        dec2.step()
    torch.cuda.synchronize()
    assert np.array_equal(dec2.history[:12].cpu().numpy(), hist)
    with pytest.raises(ValueError):
        dec.generate(SMALL.max_len + 1)
    w.close()
