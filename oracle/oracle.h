/*
 * TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * fp32 CPU restatement of the hybrid-batch forward (liboracle.so). The
 * reference has no numeric forward ("No token content, no sampling/logits",
 * reference SPEC.md:93; model execution out of scope), so this
 * oracle follows the standard Llama decoder definition (pre-RMSNorm, RoPE
 * rotate-half, GQA, SwiGLU) over the reference's batch semantics
 * (BatchEntry positions, core.cpp:42-63; KV growth, engine.cpp:211-216).
 * Parity of logits is therefore UNPINNED BY THE REFERENCE; the oracle itself
 * is pinned against an independent implementation (HF transformers
 * LlamaForCausalLM, fp32) by tests/golden/make_hf_golden.py.
 *
 * Weights, cached KV and token ids come from include/ss_synth.h (identical to
 * the GPU initialiser); the tensor-parallel shard math is the same Megatron
 * split as the GPU path, with an all-reduce callback supplied by the caller
 * (tests drive it over torch.distributed gloo).
 */
#ifndef SS_ORACLE_H
#define SS_ORACLE_H

#include <stdint.h>

#include "../include/ss_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc orc;
typedef void (*orc_allreduce_fn)(float* buf, int64_t n, void* user);

/* layers: number of decoder layers to materialise (<= cfg->num_layers; the
 * residual scaling still uses cfg->num_layers). with_head: build the LM head. */
orc* orc_create(const ss_model_cfg* cfg, int32_t tp_rank, int32_t tp_size, uint64_t weight_seed,
                int64_t num_blocks, int32_t layers, int32_t with_head);
void orc_destroy(orc* o);
void orc_set_allreduce(orc* o, orc_allreduce_fn fn, void* user);
int32_t orc_threads(void);
/* Same contract as ss_kv_fill_synthetic. */
int32_t orc_kv_fill_synthetic(orc* o, const int32_t* block_table, int32_t n_blocks, int32_t rid,
                              int32_t n_tokens, uint64_t seed);
/* Forward of one batch. logits: [n_out][vocab/tp] (this rank's vocab slice),
 * nullable. hidden: [T][hidden] final residual stream (pre final norm), nullable. */
int32_t orc_forward(orc* o, const ss_batch_desc* d, float* logits, float* hidden);
/* Copies a materialised weight ([rows][cols], fp32) for tests: names as in
 * ss_weight_ptr but unfused: "wq","wk","wv","wo","wg","wu","wd","embed","lm_head", and the
 * RMSNorm gains "attn_norm","mlp_norm" (per layer), "final_norm" ([1][hidden]). */
int32_t orc_weight(orc* o, const char* name, int32_t layer, float* out, int64_t* rows, int64_t* cols);
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
