"""Decode chain of sparse linears (BASELINE.json config 4) on cuda:0.

A reduced-size chain (2 layers, H = 256, I = 688) checked SpMV by SpMV against the oracle's
emulation of the kernel order, and the PDL-launched / CUDA-graph-captured chain checked bit-identical
to plain stream launches at full Llama2-7B layer shapes (one layer).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2511_13061_b200 import decoder_chain as D
from paper_2511_13061_b200 import macko as M
from tests.helpers import b200_y, to_host_u16

pytestmark = pytest.mark.gpu


def _h0(chain, seed=77):
    M.gen_vector(chain.acts["h"], chain.shape.hidden, seed=seed)
    chain.acts["h"].mul_(2.0**-10)  # keeps the random-weight chain inside fp16 range


def test_chain_matches_oracle(cuda):
    shape = D.ChainShape(layers=2, hidden=256, inter=688)
    seed = 1000
    ch = D.SparseDecoderChain(shape, density=0.5, seed=seed)
    _h0(ch)
    h = to_host_u16(ch.acts["h"])
    ch.forward_token(pdl=False)
    torch.cuda.synchronize()
    H, I = shape.hidden, shape.inter
    for layer in range(shape.layers):
        ws = {}
        for name in D.LINEARS:
            R, C = shape.shape(name)
            ws[name] = O.encode_dense(O.gen_dense(R, C, 0.5, D.weight_seed(seed, layer, name)))
        qkv = b200_y(ws["qkv"], h)
        o = b200_y(ws["o"], qkv[:H])  # v = first H rows of [W_v; W_q; W_k]
        gu = b200_y(ws["gate_up"], o)
        h = b200_y(ws["down"], gu[:I])  # up = first I rows of [W_up; W_gate]
    assert np.isfinite(h.view(np.float16).astype(np.float32)).all()
    assert np.array_equal(to_host_u16(ch.acts["h"]), h)
    ch.close()


def test_chain_pdl_graph_bit_identical(cuda):
    ch = D.SparseDecoderChain(D.ChainShape(layers=1, hidden=4096, inter=11008), density=0.5, seed=5)
    assert ch.kernels_per_token == 4
    _h0(ch, 3)
    h0 = ch.acts["h"].clone()
    ch.forward_token(pdl=False)
    torch.cuda.synchronize()
    ref = {k: to_host_u16(v) for k, v in ch.acts.items()}
    for pdl in (True, False):
        ch.acts["h"].copy_(h0)
        ch.forward_token(pdl=pdl)
        torch.cuda.synchronize()
        for k, v in ch.acts.items():
            assert np.array_equal(to_host_u16(v), ref[k]), (pdl, k)
    g = ch.capture(pdl=True)  # capture runs one warm-up token: reset h afterwards
    for _ in range(2):
        ch.acts["h"].copy_(h0)
        g.replay()
        torch.cuda.synchronize()
        for k, v in ch.acts.items():
            assert np.array_equal(to_host_u16(v), ref[k]), ("graph", k)
    ch.close()


