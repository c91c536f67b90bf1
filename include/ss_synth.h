/*
 * ss_synth.h — counter-based synthetic inputs shared by the GPU path and the
 * CPU oracle: random-init weights, synthetic cached KV and synthetic token ids.
 *
 * The reference carries no weights and no token content ("No token content, no
 * sampling/logits, no vocabulary", reference SPEC.md:93), so these are the
 * framework's own input definition. Every value is a pure function of
 * (seed, tag, global row, global column) and involves only integer hashing and
 * one correctly-rounded fp32 multiply, so tensor-parallel shards, the GPU
 * initialiser and the oracle produce bit-identical bf16 values.
 */
#ifndef SS_SYNTH_H
#define SS_SYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define SS_HD __host__ __device__ __forceinline__
#else
#define SS_HD static inline
#endif

/* tensor ids inside a layer */
enum { SS_T_Q = 0, SS_T_K = 1, SS_T_V = 2, SS_T_O = 3, SS_T_GATE = 4, SS_T_UP = 5, SS_T_DOWN = 6 };
#define SS_TAG_LAYER(l, t) (0x100u + (uint32_t)(l) * 16u + (uint32_t)(t))
#define SS_TAG_EMBED 0xE0000u
#define SS_TAG_LMHEAD 0xE0001u
#define SS_TAG_TOKEN 0xA0000u
#define SS_TAG_KV(l, which) (0xC0000u + (uint32_t)(l) * 2u + (uint32_t)(which))
/* RMSNorm gains: which = 0 attn_norm (input_layernorm), 1 mlp_norm (post-attention), 2 final */
enum { SS_NORM_ATTN = 0, SS_NORM_MLP = 1, SS_NORM_FINAL = 2 };
#define SS_TAG_NORM(l, which) (0xD0000u + (uint32_t)(l) * 4u + (uint32_t)(which))

SS_HD uint64_t ss_mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

SS_HD uint64_t ss_key(uint64_t seed, uint32_t tag, uint64_t a, uint64_t b) {
    return ss_mix64(ss_mix64(seed ^ (0x9E3779B97F4A7C15ull * ((uint64_t)tag + 1ull))) ^
                    ss_mix64(a * 0xD1B54A32D192ED03ull + b));
}

/* Uniform in [-1, 1) with 24 significant bits (exact in fp32). */
SS_HD float ss_unit(uint64_t h) {
    return (float)((int32_t)(h >> 40) - (int32_t)(1 << 23)) * (1.0f / 8388608.0f);
}

/* fp32 -> bf16 bits, round to nearest even (inputs are finite). */
SS_HD uint16_t ss_f32_to_bf16_bits(float f) {
    union {
        float f;
        uint32_t u;
    } v;
    v.f = f;
    uint32_t b = v.u;
    b += 0x7FFFu + ((b >> 16) & 1u);
    return (uint16_t)(b >> 16);
}

SS_HD float ss_bf16_bits_to_f32(uint16_t h) {
    union {
        float f;
        uint32_t u;
    } v;
    v.u = ((uint32_t)h) << 16;
    return v.f;
}

/* bf16 bits of element (row, col) of a tensor with per-tensor scale. */
SS_HD uint16_t ss_synth_bf16(uint64_t seed, uint32_t tag, uint64_t row, uint64_t col, float scale) {
    return ss_f32_to_bf16_bits(ss_unit(ss_key(seed, tag, row, col)) * scale);
}

/* RMSNorm gain element i (bf16 bits): 1 + u/4, u uniform in [-1, 1), so gains lie in
 * [0.75, 1.25) — non-unit, so a dropped or misapplied gain changes every logit. The
 * product u/4 is exact; the sum is one correctly-rounded fp32 add (FMA-safe). */
SS_HD uint16_t ss_norm_gain_bf16(uint64_t seed, int layer, int which, int64_t i) {
    return ss_f32_to_bf16_bits(1.0f + 0.25f * ss_unit(ss_key(seed, SS_TAG_NORM(layer, which), 0u, (uint64_t)i)));
}

/* Synthetic token id of request rid at absolute position pos. */
SS_HD int32_t ss_token_id(uint64_t seed, int64_t rid, int64_t pos, int32_t vocab) {
    return (int32_t)(ss_key(seed, SS_TAG_TOKEN, (uint64_t)rid, (uint64_t)pos) % (uint64_t)vocab);
}

/* Synthetic cached K (which=0) / V (which=1) value of request rid at position
 * pos, global kv head kvh, dim d; unit variance. */
SS_HD uint16_t ss_synth_kv(uint64_t seed, int layer, int which, int64_t rid, int64_t pos,
                           int kvh, int d, int num_kv_heads, int head_dim) {
    return ss_synth_bf16(seed, SS_TAG_KV(layer, which), (uint64_t)rid,
                         ((uint64_t)pos * (uint64_t)num_kv_heads + (uint64_t)kvh) *
                                 (uint64_t)head_dim + (uint64_t)d,
                         1.7320508075688772f);
}

#include <math.h>
/* Per-tensor scale: uniform[-s, s) has variance s^2/3, so s = sqrt(3/fan_in)
 * gives N(0, 1/fan_in)-matched variance; O and down projections are further
 * scaled by 1/sqrt(2L) so the residual stream stays O(1) over L layers.
 * Embeddings have unit variance. Computed in double, rounded once to fp32. */
static inline float ss_weight_scale(int tensor_id, int64_t fan_in, int num_layers) {
    double s = sqrt(3.0 / (double)fan_in);
    if (tensor_id == SS_T_O || tensor_id == SS_T_DOWN) s /= sqrt(2.0 * (double)num_layers);
    return (float)s;
}
static inline float ss_embed_scale(void) { return 1.7320508075688772f; }
/* RoPE (rotate-half, HF Llama convention) table entry for position p and
 * pair index i < hd/2: angle = p * theta^(-2i/hd), evaluated in double and
 * rounded once; the GPU path and the oracle share these exact values. */
static inline void ss_rope_cs(double theta, int hd, int64_t p, int i, float* c, float* s) {
    const double inv = pow(theta, -2.0 * (double)i / (double)hd);
    const double a = (double)p * inv;
    *c = (float)cos(a);
    *s = (float)sin(a);
}

#endif /* SS_SYNTH_H */
