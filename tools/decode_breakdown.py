"""Where the Llama2-7B decode step's time goes (CUDA graphs, CUDA events): the full MACKO step, the
same step without the per-token kernels (SpMVs + LM head only), the per-token kernels alone, and
the dense (cuBLAS) step / its GEMVs alone."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13061_b200 import llama as L  # noqa: E402

torch.cuda.set_device(0)
w = L.LlamaWeights(L.LLAMA2_7B, density=0.5)


def graph_ms(fn, n=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn(s)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n


for kind in ("macko", "dense"):
    d = L.LlamaDecoder(w, kind)
    d.reset()
    full = graph_ms(lambda s: d.step(s, sample=False))
    for pos in (50, 99):
        d.pos.fill_(pos)
        print(f"  {kind} step at position {pos}: {graph_ms(lambda s: d.step(s, sample=False)):.3f} ms", flush=True)
    d.pos.fill_(0)
    print(f"  {kind} step with argmax: {graph_ms(lambda s: d.step(s, sample=True)):.3f} ms", flush=True)

    def linears_only(s):
        for layer in range(d.cfg.layers):
            d._linear(layer, "qkv", d.x, d.qkv, s)
            d._linear(layer, "o", d.attn, d.delta, s)
            d._linear(layer, "gate_up", d.x, d.gu, s)
            d._linear(layer, "down", d.act, d.delta, s)
    lin = graph_ms(linears_only)

    def small_only(s):
        Lb, cfg = L.llm_lib(), d.cfg
        p = lambda t: t.data_ptr()  # noqa: E731
        ss = s.cuda_stream
        for layer in range(cfg.layers):
            nrm = w.norms[layer]
            Lb.macko_llm_add_rmsnorm(p(d.h), p(d.delta) if layer else None, p(nrm["ln1"]), p(d.x), cfg.hidden, cfg.eps, ss)
            Lb.macko_llm_rope_attention(p(d.qkv), p(d.pos), p(d.k_cache[layer]), p(d.v_cache[layer]), p(d.attn),
                                        cfg.heads, cfg.head_dim, cfg.max_len, cfg.theta, ss)
            Lb.macko_llm_add_rmsnorm(p(d.h), p(d.delta), p(nrm["ln2"]), p(d.x), cfg.hidden, cfg.eps, ss)
            Lb.macko_llm_silu_mul(p(d.gu), p(d.act), cfg.inter, ss)
    sm = graph_ms(small_only)
    print(f"{kind}: full step {full:.3f} ms, linears only {lin:.3f} ms, per-token kernels only {sm:.3f} ms", flush=True)
