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
    order = ch.mats[0]["qkv"].order
    for layer in range(shape.layers):
        ws = {}
        for name in D.LINEARS:
            R, C = shape.shape(name)
            ws[name] = O.encode_dense(O.gen_dense(R, C, 0.5, D.weight_seed(seed, layer, name)))
        qkv = b200_y(order, ws["qkv"], h)
        o = b200_y(order, ws["o"], qkv[:H])  # v = first H rows of [W_v; W_q; W_k]
        gu = b200_y(order, ws["gate_up"], o)
        h = b200_y(order, ws["down"], gu[:I])  # up = first I rows of [W_up; W_gate]
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


def test_persistent_chain_bit_identical(cuda):
    # one cooperative kernel per token (grid barrier between dependent SpMVs) == op-by-op launches,
    # over several tokens (the activations are rewritten inside the launch: x staging and the
    # texture gathers must never see stale lines)
    for shape in (D.ChainShape(layers=2, hidden=4096, inter=11008), D.ChainShape(layers=3, hidden=256, inter=688)):
        ch = D.SparseDecoderChain(shape, density=0.5, seed=9)
        _h0(ch, 4)
        h0 = ch.acts["h"].clone()
        refs = []
        for _ in range(3):
            ch.forward_token(pdl=False)
            torch.cuda.synchronize()
            refs.append({k: to_host_u16(v) for k, v in ch.acts.items()})
        ch.acts["h"].copy_(h0)
        for tok in range(3):
            ch.forward_token_persistent()
            torch.cuda.synchronize()
            for k, v in ch.acts.items():
                assert np.array_equal(to_host_u16(v), refs[tok][k]), (shape, tok, k)
        # CUDA-graph capture of the persistent launch
        s = torch.cuda.Stream()
        ch.acts["h"].copy_(h0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ch.forward_token_persistent(s)
        ch.acts["h"].copy_(h0)
        for tok in range(2):
            g.replay()
            torch.cuda.synchronize()
            assert np.array_equal(to_host_u16(ch.acts["h"]), refs[tok]["h"]), ("graph", shape, tok)
        ch.close()


def test_persistent_chain_rejects_flat_walk(cuda):
    # the cooperative chain kernel runs the ROMA walk only; a flat-walk matrix is refused
    ch = D.SparseDecoderChain(D.ChainShape(layers=1, hidden=256, inter=688), density=0.5, seed=3)
    ch.mats[0]["o"].set_order(1)
    with pytest.raises(ValueError):
        ch.persistent()
    ch.close()


def test_chain_create_rejects_bad_ops(cuda):
    # b_delta != 4 and a misaligned x are refused; a valid one-op chain equals macko_dev_spmv
    w = torch.empty((512, 1024), dtype=torch.float16, device=cuda)
    M.gen_dense(w, 512, 1024, 0.5, seed=1)
    dm8 = M.DeviceMatrix.from_dense(w, b_delta=8)
    dm4 = M.DeviceMatrix.from_dense(w)
    buf = torch.zeros(4096, dtype=torch.float16, device=cuda)
    y = torch.zeros(512, dtype=torch.float16, device=cuda)
    with pytest.raises(ValueError):
        M.Chain([(dm8, buf[:1024], y)])
    with pytest.raises(ValueError):
        M.Chain([(dm4, buf[1:1025], y)])  # 2-byte aligned only: the chain stages x without a copy
    ch = M.Chain([(dm4, buf[:1024], y)])
    ch.run()
    torch.cuda.synchronize()
    ref = M.spmv(dm4, buf[:1024])
    assert torch.equal(ref, y)
    ch.close()
    dm8.close()
    dm4.close()
