/*
 * macko_llm.h — libmacko_llm.so: per-token kernels of a Llama-style batch-1 decode step (the caller
 * of the MACKO SpMV in the paper's end-to-end benchmark).  fp16 tensors as raw
 * uint16 bits, device pointers, `stream` a cudaStream_t (NULL = legacy default).  Positions and
 * token ids live in device memory so a decode step is graph-capturable.  Returns cudaError_t.
 */
#ifndef MACKO_LLM_H
#define MACKO_LLM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* h += delta (if delta != NULL, fp16 residual); out = h * rsqrt(mean(h^2) + eps) * weight (RMSNorm). */
int macko_llm_add_rmsnorm(uint16_t* h, const uint16_t* delta, const uint16_t* weight, uint16_t* out, uint32_t n,
                          float eps, void* stream);
/* qkv = [q; k; v]: rotary embedding (rotate-half, base theta) of q and k at position *pos, k / v appended
 * to cache row *pos (heads * head_dim each), then multi-head attention of the rotated q over cache rows
 * [0, *pos] (fp32 softmax) into out.  One CTA per head. */
int macko_llm_rope_attention(const uint16_t* qkv, const int32_t* pos, uint16_t* k_cache, uint16_t* v_cache,
                             uint16_t* out, uint32_t heads, uint32_t head_dim, uint32_t max_len, float theta,
                             void* stream);
/* gu = [gate; up]: out = silu(gate) * up. */
int macko_llm_silu_mul(const uint16_t* gu, uint16_t* out, uint32_t inter, void* stream);
/* h = table[*token]. */
int macko_llm_embed(const uint16_t* table, const int32_t* token, uint16_t* h, uint32_t hidden, void* stream);
/* *token = argmax(logits) (lowest index on ties); history[*pos] = *token; *pos += 1. */
int macko_llm_argmax(const uint16_t* logits, uint32_t n, int32_t* token, int32_t* pos, int32_t* history,
                     uint32_t history_len, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MACKO_LLM_H */
