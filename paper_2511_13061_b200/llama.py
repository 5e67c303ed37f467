"""Llama2-7B batch-1 greedy decode with MACKO linears vs dense cuBLAS linears — the paper's
end-to-end measurement (Llama2-7B pruned to 50 %, 100 tokens generated from an
empty prompt, tokens/s of the dense model vs the same weights in MACKO).

Random-init weights (no checkpoints here): every decoder linear is a Bernoulli(density) mask of the
counter-hash generator's uniform [-1, 1) values, scaled so activations stay O(1); the embedding, the
norms and the LM head stay dense, as in the paper (the pruner does not touch them).
Both variants use the SAME pruned fp16 weights: the MACKO model compresses exactly the matrices the
dense model multiplies with cuBLAS (MACKO is lossless), so they differ only by fp32 summation order.

A decode step (per layer: RMSNorm -> qkv -> RoPE + KV append + attention -> o -> add + RMSNorm ->
gate_up -> SiLU * up -> down, then the final norm, the LM head and greedy argmax) reads its position
and token from device memory, so one CUDA graph replays token after token.  The per-token kernels
are libmacko_llm.so (csrc/llm.cu); q/k/v and gate/up are row-stacked into one matrix each (rows are
independent: the stacked MACKO encoding is the concatenation of the encodings).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass
from typing import Dict, List, Optional

import torch

from . import macko as M
from .decoder_chain import CHAIN_SKEW_NS

HERE = os.path.dirname(os.path.abspath(__file__))
_llm = None


def llm_lib() -> C.CDLL:
    global _llm
    if _llm is None:
        path = os.path.join(HERE, "libmacko_llm.so")
        if not os.path.exists(path):
            raise OSError(f"libmacko_llm.so not built at {path}; run `make llm`")
        L = C.CDLL(path)
        vp, u32, i = C.c_void_p, C.c_uint32, C.c_int
        for name, args in {
            "macko_llm_add_rmsnorm": [vp, vp, vp, vp, u32, C.c_float, vp],
            "macko_llm_rope_attention": [vp, vp, vp, vp, vp, u32, u32, u32, C.c_float, vp],
            "macko_llm_silu_mul": [vp, vp, u32, vp],
            "macko_llm_embed": [vp, vp, vp, u32, vp],
            "macko_llm_argmax": [vp, u32, vp, vp, vp, u32, vp],
        }.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = i
        _llm = L
    return _llm


def _ck(rc: int, what: str) -> None:
    if rc != 0:
        raise RuntimeError(f"{what}: cudaError {rc}")


@dataclass(frozen=True)
class LlamaConfig:
    vocab: int = 32000
    hidden: int = 4096
    layers: int = 32
    heads: int = 32
    inter: int = 11008
    max_len: int = 128
    eps: float = 1e-5
    theta: float = 10000.0

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


LLAMA2_7B = LlamaConfig()
LINEARS = ("qkv", "o", "gate_up", "down")


def linear_shape(cfg: LlamaConfig, name: str):
    H, I = cfg.hidden, cfg.inter
    return {"qkv": (3 * H, H), "o": (H, H), "gate_up": (2 * I, H), "down": (H, I)}[name]


def _gen(shape, density, seed, scale, device):
    w = torch.empty(shape, dtype=torch.float16, device=device)
    M.gen_dense(w, shape[0], shape[1], density, seed=seed)
    w.mul_(scale)
    return w


class LlamaWeights:
    """Random-init, pruned Llama weights; per layer the linears as dense fp16 tensors and/or MACKO
    matrices compressed on the GPU from exactly those tensors."""

    def __init__(self, cfg: LlamaConfig = LLAMA2_7B, density: float = 0.5, seed: int = 0x11A3A,
                 device: Optional[torch.device] = None, keep_dense: bool = True, macko: bool = True):
        self.cfg, self.density = cfg, density
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        H = cfg.hidden
        self.embed = _gen((cfg.vocab, H), 1.0, seed, 1.0, dev)
        self.lm_head = _gen((cfg.vocab, H), 1.0, seed + 1, math.sqrt(3.0 / H), dev)
        self.norm_f = torch.ones(H, dtype=torch.float16, device=dev)
        self.dense: List[Dict[str, torch.Tensor]] = []
        self.mats: List[Dict[str, M.DeviceMatrix]] = []
        self.norms: List[Dict[str, torch.Tensor]] = []
        for layer in range(cfg.layers):
            dl, ml = {}, {}
            for k, name in enumerate(LINEARS):
                R, Cc = linear_shape(cfg, name)
                # var(y) ~ 1 for unit-rms inputs: uniform[-1,1) has variance 1/3 over density*C terms
                w = _gen((R, Cc), density, seed + 100 + 16 * layer + k, math.sqrt(3.0 / (density * Cc)), dev)
                if macko:
                    ml[name] = M.DeviceMatrix.from_dense(w)
                    if CHAIN_SKEW_NS:  # every decode-step SpMV is a PDL dependent (decoder_chain.py)
                        ml[name].set_chain_skew(CHAIN_SKEW_NS)
                if keep_dense:
                    dl[name] = w
                else:
                    del w
            self.dense.append(dl)
            self.mats.append(ml)
            self.norms.append({"ln1": torch.ones(H, dtype=torch.float16, device=dev),
                               "ln2": torch.ones(H, dtype=torch.float16, device=dev)})
        torch.cuda.synchronize(dev)

    @property
    def macko_bytes(self) -> int:
        return sum(m.info.values_bytes + m.info.delta_bytes + m.info.row_ptr_bytes
                   for ml in self.mats for m in ml.values())

    @property
    def dense_bytes(self) -> int:
        return sum(2 * w.numel() for dl in self.dense for w in dl.values())

    def close(self) -> None:
        for ml in self.mats:
            for m in ml.values():
                m.close()
        self.mats, self.dense = [], []


class LlamaDecoder:
    """One decode step of the model with `linears` = "macko" (libmacko_cuda SpMVs, PDL-chained) or
    "dense" (torch.mv = cuBLAS GEMV) over the same weights; greedy argmax feeds the next token."""

    def __init__(self, w: LlamaWeights, linears: str = "macko"):
        if linears not in ("macko", "dense"):
            raise ValueError("linears must be 'macko' or 'dense'")
        if linears == "macko" and not w.mats[0]:
            raise ValueError("weights were built without MACKO matrices")
        if linears == "dense" and not w.dense[0]:
            raise ValueError("weights were built without dense tensors")
        self.w, self.cfg, self.linears = w, w.cfg, linears
        cfg, dev = w.cfg, w.device
        H, I = cfg.hidden, cfg.inter
        z = lambda n: torch.zeros(n, dtype=torch.float16, device=dev)  # noqa: E731
        self.h, self.x, self.delta = z(H), z(H), z(H)
        self.qkv, self.attn = z(3 * H), z(H)
        self.gu, self.act, self.logits = z(2 * I), z(I), z(cfg.vocab)
        self.k_cache = torch.zeros((cfg.layers, cfg.max_len, H), dtype=torch.float16, device=dev)
        self.v_cache = torch.zeros_like(self.k_cache)
        self.pos = torch.zeros(1, dtype=torch.int32, device=dev)
        self.token = torch.ones(1, dtype=torch.int32, device=dev)  # BOS = 1
        self.history = torch.zeros(cfg.max_len, dtype=torch.int32, device=dev)
        self.graph: Optional[torch.cuda.CUDAGraph] = None

    def reset(self, token: int = 1) -> None:
        self.pos.zero_()
        self.token.fill_(token)
        self.history.zero_()
        self.k_cache.zero_()
        self.v_cache.zero_()

    def _linear(self, layer: int, name: str, x: torch.Tensor, y: torch.Tensor, stream) -> None:
        if self.linears == "macko":
            self.w.mats[layer][name].spmv_into(x, y, stream, pdl=True)
        else:
            torch.mv(self.w.dense[layer][name], x, out=y)

    def step(self, stream=None, sample: bool = True) -> None:
        """One token (stream-ordered): logits of the token at *pos, then (sample) argmax -> token, pos + 1."""
        L, cfg = llm_lib(), self.cfg
        s = (stream if stream is not None else torch.cuda.current_stream()).cuda_stream
        p = lambda t: t.data_ptr()  # noqa: E731
        H, I = cfg.hidden, cfg.inter
        st = stream if stream is not None else torch.cuda.current_stream()
        _ck(L.macko_llm_embed(p(self.w.embed), p(self.token), p(self.h), H, s), "embed")
        for layer in range(cfg.layers):
            nrm = self.w.norms[layer]
            _ck(L.macko_llm_add_rmsnorm(p(self.h), p(self.delta) if layer else None, p(nrm["ln1"]), p(self.x), H,
                                        cfg.eps, s), "rmsnorm")
            self._linear(layer, "qkv", self.x, self.qkv, st)
            _ck(L.macko_llm_rope_attention(p(self.qkv), p(self.pos), p(self.k_cache[layer]), p(self.v_cache[layer]),
                                           p(self.attn), cfg.heads, cfg.head_dim, cfg.max_len, cfg.theta, s),
                "rope_attention")
            self._linear(layer, "o", self.attn, self.delta, st)
            _ck(L.macko_llm_add_rmsnorm(p(self.h), p(self.delta), p(nrm["ln2"]), p(self.x), H, cfg.eps, s),
                "rmsnorm")
            self._linear(layer, "gate_up", self.x, self.gu, st)
            _ck(L.macko_llm_silu_mul(p(self.gu), p(self.act), I, s), "silu")
            self._linear(layer, "down", self.act, self.delta, st)
        _ck(L.macko_llm_add_rmsnorm(p(self.h), p(self.delta), p(self.w.norm_f), p(self.x), H, cfg.eps, s), "rmsnorm")
        torch.mv(self.w.lm_head, self.x, out=self.logits)
        if sample:
            _ck(L.macko_llm_argmax(p(self.logits), cfg.vocab, p(self.token), p(self.pos), p(self.history),
                                   cfg.max_len, s), "argmax")

    def capture(self) -> torch.cuda.CUDAGraph:
        """One decode step as a CUDA graph (warm-up on the capture stream first)."""
        s = torch.cuda.Stream(device=self.w.device)
        s.wait_stream(torch.cuda.current_stream(self.w.device))
        with torch.cuda.stream(s):
            self.step(s)  # warm-up: SpMV workspaces / texture objects for this stream, cuBLAS handles
        torch.cuda.current_stream(self.w.device).wait_stream(s)
        torch.cuda.synchronize(self.w.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.step(s)
        self.graph = g
        return g

    def generate(self, n: int) -> float:
        """Greedy-decode n tokens from BOS with the captured step; returns seconds (CUDA events)."""
        if n > self.cfg.max_len:
            raise ValueError("n exceeds max_len")
        g = self.graph or self.capture()
        self.reset()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            g.replay()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) * 1e-3


def bench_decode(torch_mod=torch, dev=None, n_tokens: int = 100, density: float = 0.5) -> dict:
    """tokens/s of Llama2-7B (random-init, 50 % unstructured) generating n_tokens from BOS: MACKO
    linears vs dense cuBLAS linears over the same weights."""
    t0 = time.time()
    w = LlamaWeights(LLAMA2_7B, density=density, device=dev)
    build_s = time.time() - t0
    out = {"model": "Llama2-7B (32 layers, hidden 4096, 32 heads, inter 11008, vocab 32000), random-init, "
                    f"decoder linears pruned to {int(round((1 - density) * 100))}% unstructured; embedding / LM head dense",
           "tokens": n_tokens, "prompt": "BOS only (empty prompt), greedy", "build_s": round(build_s, 1),
           "macko_linear_GB": round(w.macko_bytes / 1e9, 3), "dense_linear_GB": round(w.dense_bytes / 1e9, 3)}
    res = {}
    for kind in ("dense", "macko"):
        d = LlamaDecoder(w, kind)
        d.capture()
        d.generate(min(8, n_tokens))  # warm-up replays
        secs = [d.generate(n_tokens) for _ in range(3)]
        sec = sorted(secs)[1]
        res[kind] = {"tokens_per_s": round(n_tokens / sec, 2), "ms_per_token": round(sec * 1e3 / n_tokens, 3),
                     "history": d.history[:n_tokens].cpu().tolist(), "logits": d.logits.float().clone()}
        del d
        torch.cuda.empty_cache()
    same = sum(int(a == b) for a, b in zip(res["dense"]["history"], res["macko"]["history"]))
    first_diverge = next((i for i, (a, b) in enumerate(zip(res["dense"]["history"], res["macko"]["history"]))
                          if a != b), None)
    out.update({"dense_tokens_per_s": res["dense"]["tokens_per_s"], "dense_ms_per_token": res["dense"]["ms_per_token"],
                "macko_tokens_per_s": res["macko"]["tokens_per_s"], "macko_ms_per_token": res["macko"]["ms_per_token"],
                "speedup": round(res["macko"]["tokens_per_s"] / res["dense"]["tokens_per_s"], 3),
                "greedy_tokens_equal": f"{same}/{n_tokens}", "first_divergent_token": first_diverge,
                "timing": "CUDA graph of one decode step replayed per token, CUDA events, median of 3 runs"})
    w.close()
    torch.cuda.empty_cache()
    return out
