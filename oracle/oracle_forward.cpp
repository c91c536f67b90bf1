// TEST INFRASTRUCTURE ONLY — see oracle.h for what this restates and how it is
// pinned. fp32 throughout: weights are the bf16-representable values of
// ss_synth.h held in fp32, activations are never rounded to bf16, softmax is
// exact (max-subtracted, fp32), matmuls accumulate in fp32.
#include "oracle.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../include/ss_synth.h"

namespace {

thread_local std::string g_err;

typedef float v16 __attribute__((vector_size(64)));

// C[M][N] (+)= A[M][K] . B[N][K]^T, row-major, fp32. Blocked for L1/L2 reuse:
// each thread owns 64-row slabs of B (the weights), walks K in 256-wide
// chunks and all of M in 4-row strips with a 4x4 register micro-kernel.
__attribute__((target_clones("avx512f", "avx2", "default"))) void micro_4x4(const float* a, int64_t lda,
                                                                           const float* b, int64_t ldb, int kc,
                                                                           int mr, int nr, float* c, int64_t ldc) {
    float acc[4][4] = {};
    if (mr == 4 && nr == 4 && kc % 16 == 0) {
        v16 s[4][4];
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) s[i][j] = v16{};
        for (int k = 0; k < kc; k += 16) {
            v16 av[4], bv[4];
            for (int i = 0; i < 4; ++i) std::memcpy(&av[i], a + i * lda + k, 64);
            for (int j = 0; j < 4; ++j) std::memcpy(&bv[j], b + j * ldb + k, 64);
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) s[i][j] += av[i] * bv[j];
        }
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) {
                float t = 0.f;
                for (int l = 0; l < 16; ++l) t += s[i][j][l];
                acc[i][j] = t;
            }
    } else {
        for (int i = 0; i < mr; ++i)
            for (int j = 0; j < nr; ++j) {
                float t = 0.f;
                for (int k = 0; k < kc; ++k) t += a[i * lda + k] * b[j * ldb + k];
                acc[i][j] = t;
            }
    }
    for (int i = 0; i < mr; ++i)
        for (int j = 0; j < nr; ++j) c[i * ldc + j] += acc[i][j];
}

void sgemm_nt(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K, bool accumulate) {
    if (!accumulate)
        for (int64_t i = 0; i < M * N; ++i) C[i] = 0.f;
    const int64_t NB = 64, KB = 256;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t nb = 0; nb < N; nb += NB) {
        const int64_t ne = std::min(N, nb + NB);
        for (int64_t kb = 0; kb < K; kb += KB) {
            const int kc = int(std::min(K, kb + KB) - kb);
            for (int64_t m = 0; m < M; m += 4) {
                const int mr = int(std::min<int64_t>(4, M - m));
                for (int64_t n = nb; n < ne; n += 4) {
                    const int nr = int(std::min<int64_t>(4, ne - n));
                    micro_4x4(A + m * K + kb, K, B + n * K + kb, K, kc, mr, nr, C + m * N + n, N);
                }
            }
        }
    }
}

struct Layer {
    std::vector<float> wq, wk, wv, wo, wg, wu, wd;  // unfused, natural layouts
    std::vector<float> g_attn, g_mlp;               // RMSNorm gains, applied explicitly
};

}  // namespace

struct orc {
    ss_model_cfg cfg;
    int rank, tp, nq, nkv, G, hd, h, ffn, vl, L;
    bool head;
    uint64_t seed;
    std::vector<Layer> layers;
    std::vector<float> embed, lm_head, g_final;
    std::vector<float> kc, vc;  // [L][nblocks][nkv][16][hd]
    int64_t nblocks, lstride;
    std::vector<float> cosv, sinv;  // [max_pos][hd/2]
    orc_allreduce_fn ar = nullptr;
    void* ar_user = nullptr;
};

namespace {

void gen(std::vector<float>& w, int64_t rows, int64_t cols, uint64_t seed, uint32_t tag, int64_t row_off,
         int64_t col_off, float scale) {
    w.resize(size_t(rows * cols));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j)
            w[size_t(i * cols + j)] = ss_bf16_bits_to_f32(
                ss_synth_bf16(seed, tag, uint64_t(row_off + i), uint64_t(col_off + j), scale));
}

// HF LlamaRMSNorm: out = g * (x * rsqrt(mean(x^2) + eps))
void rmsnorm_rows(const float* x, const float* g, float* out, int64_t M, int64_t h, float eps) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < M; ++r) {
        double ss = 0;
        for (int64_t i = 0; i < h; ++i) ss += double(x[r * h + i]) * x[r * h + i];
        const float inv = float(1.0 / std::sqrt(ss / double(h) + double(eps)));
        for (int64_t i = 0; i < h; ++i) out[r * h + i] = g[i] * (x[r * h + i] * inv);
    }
}

void gen_gain(std::vector<float>& g, int64_t h, uint64_t seed, int layer, int which) {
    g.resize(size_t(h));
    for (int64_t i = 0; i < h; ++i) g[size_t(i)] = ss_bf16_bits_to_f32(ss_norm_gain_bf16(seed, layer, which, i));
}

void allreduce(orc* o, float* buf, int64_t n) {
    if (o->tp > 1 && o->ar) o->ar(buf, n, o->ar_user);
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int32_t orc_threads(void) { return omp_get_max_threads(); }

orc* orc_create(const ss_model_cfg* cfg, int32_t tp_rank, int32_t tp_size, uint64_t seed, int64_t num_blocks,
                int32_t layers, int32_t with_head) {
    if (!cfg || tp_size < 1 || cfg->num_q_heads % tp_size || cfg->num_kv_heads % tp_size || cfg->ffn % tp_size ||
        cfg->vocab % tp_size || layers < 0 || layers > cfg->num_layers || num_blocks < 1) {
        g_err = "bad oracle configuration";
        return nullptr;
    }
    orc* o = new orc();
    o->cfg = *cfg;
    o->rank = tp_rank;
    o->tp = tp_size;
    o->nq = cfg->num_q_heads / tp_size;
    o->nkv = cfg->num_kv_heads / tp_size;
    o->G = o->nq / o->nkv;
    o->hd = cfg->head_dim;
    o->h = cfg->hidden;
    o->ffn = cfg->ffn / tp_size;
    o->vl = cfg->vocab / tp_size;
    o->L = layers;
    o->head = with_head != 0;
    o->seed = seed;
    const int64_t h = o->h, hd = o->hd, Lg = cfg->num_layers;
    const float sq = ss_weight_scale(SS_T_Q, h, int(Lg));
    const float so = ss_weight_scale(SS_T_O, int64_t(cfg->num_q_heads) * hd, int(Lg));
    const float sd = ss_weight_scale(SS_T_DOWN, cfg->ffn, int(Lg));
    o->layers.resize(size_t(layers));
    for (int l = 0; l < layers; ++l) {
        Layer& W = o->layers[size_t(l)];
        const int64_t qr = int64_t(o->nq) * hd, kr = int64_t(o->nkv) * hd;
        gen(W.wq, qr, h, seed, SS_TAG_LAYER(l, SS_T_Q), tp_rank * qr, 0, sq);
        gen(W.wk, kr, h, seed, SS_TAG_LAYER(l, SS_T_K), tp_rank * kr, 0, sq);
        gen(W.wv, kr, h, seed, SS_TAG_LAYER(l, SS_T_V), tp_rank * kr, 0, sq);
        gen(W.wo, h, qr, seed, SS_TAG_LAYER(l, SS_T_O), 0, tp_rank * qr, so);
        gen(W.wg, o->ffn, h, seed, SS_TAG_LAYER(l, SS_T_GATE), int64_t(tp_rank) * o->ffn, 0, sq);
        gen(W.wu, o->ffn, h, seed, SS_TAG_LAYER(l, SS_T_UP), int64_t(tp_rank) * o->ffn, 0, sq);
        gen(W.wd, h, o->ffn, seed, SS_TAG_LAYER(l, SS_T_DOWN), 0, int64_t(tp_rank) * o->ffn, sd);
        gen_gain(W.g_attn, h, seed, l, SS_NORM_ATTN);
        gen_gain(W.g_mlp, h, seed, l, SS_NORM_MLP);
    }
    gen_gain(o->g_final, h, seed, 0, SS_NORM_FINAL);
    gen(o->embed, cfg->vocab, h, seed, SS_TAG_EMBED, 0, 0, ss_embed_scale());
    if (o->head) gen(o->lm_head, o->vl, h, seed, SS_TAG_LMHEAD, int64_t(tp_rank) * o->vl, 0, sq);
    o->nblocks = num_blocks;
    o->lstride = num_blocks * o->nkv * 16 * hd;
    o->kc.assign(size_t(o->lstride) * size_t(std::max(layers, 1)), 0.f);
    o->vc.assign(size_t(o->lstride) * size_t(std::max(layers, 1)), 0.f);
    const int half = int(hd / 2);
    o->cosv.resize(size_t(cfg->max_positions) * half);
    o->sinv.resize(size_t(cfg->max_positions) * half);
    for (int64_t p = 0; p < cfg->max_positions; ++p)
        for (int i = 0; i < half; ++i)
            ss_rope_cs(double(cfg->rope_theta), int(hd), p, i, &o->cosv[size_t(p * half + i)],
                       &o->sinv[size_t(p * half + i)]);
    return o;
}

void orc_destroy(orc* o) { delete o; }

void orc_set_allreduce(orc* o, orc_allreduce_fn fn, void* user) {
    o->ar = fn;
    o->ar_user = user;
}

int32_t orc_kv_fill_synthetic(orc* o, const int32_t* bt, int32_t n_blocks, int32_t rid, int32_t n_tokens,
                              uint64_t seed) {
    if (int64_t(n_blocks) * 16 < n_tokens) return 1;
#pragma omp parallel for collapse(2) schedule(static)
    for (int l = 0; l < o->L; ++l)
        for (int pos = 0; pos < n_tokens; ++pos)
            for (int h = 0; h < o->nkv; ++h)
                for (int d = 0; d < o->hd; ++d) {
                    const int64_t off = l * o->lstride + ((int64_t(bt[pos / 16]) * o->nkv + h) * 16 + pos % 16) * o->hd + d;
                    const int kvh = o->rank * o->nkv + h;
                    o->kc[size_t(off)] = ss_bf16_bits_to_f32(
                        ss_synth_kv(seed, l, 0, rid, pos, kvh, d, o->cfg.num_kv_heads, o->hd));
                    o->vc[size_t(off)] = ss_bf16_bits_to_f32(
                        ss_synth_kv(seed, l, 1, rid, pos, kvh, d, o->cfg.num_kv_heads, o->hd));
                }
    return 0;
}

int32_t orc_forward(orc* o, const ss_batch_desc* d, float* logits, float* hidden) {
    const int64_t T = d->num_tokens, E = d->num_entries, h = o->h, hd = o->hd;
    const int64_t qr = int64_t(o->nq) * hd, kr = int64_t(o->nkv) * hd;
    const int half = int(hd / 2);
    const float eps = o->cfg.rms_eps;
    for (int64_t t = 0; t < T; ++t)
        if (d->slot[t] / 16 >= o->nblocks) {
            g_err = "slot outside the oracle KV pool";
            return 2;
        }
    std::vector<float> x(size_t(T * h)), xn(size_t(T * h)), q(size_t(T * qr)), k(size_t(T * kr)), v(size_t(T * kr)),
        att(size_t(T * qr)), part(size_t(T * h)), g(size_t(T * o->ffn)), u(size_t(T * o->ffn));
    for (int64_t t = 0; t < T; ++t)
        std::memcpy(&x[size_t(t * h)], &o->embed[size_t(int64_t(d->token_ids[t]) * h)], size_t(h) * 4);
    // token -> entry map
    std::vector<int> ent(static_cast<size_t>(T));
    for (int64_t e = 0; e < E; ++e)
        for (int t = d->cu_q[e]; t < d->cu_q[e + 1]; ++t) ent[size_t(t)] = int(e);

    for (int l = 0; l < o->L; ++l) {
        const Layer& W = o->layers[size_t(l)];
        float* KC = &o->kc[size_t(l * o->lstride)];
        float* VC = &o->vc[size_t(l * o->lstride)];
        rmsnorm_rows(x.data(), W.g_attn.data(), xn.data(), T, h, eps);
        sgemm_nt(xn.data(), W.wq.data(), q.data(), T, qr, h, false);
        sgemm_nt(xn.data(), W.wk.data(), k.data(), T, kr, h, false);
        sgemm_nt(xn.data(), W.wv.data(), v.data(), T, kr, h, false);
        // RoPE (rotate-half) on q and k; append k, v at slot[t]
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < T; ++t) {
            const int64_t p = d->pos[t];
            const float* cs = &o->cosv[size_t(p * half)];
            const float* sn = &o->sinv[size_t(p * half)];
            auto rot = [&](float* r) {
                for (int i = 0; i < half; ++i) {
                    const float a = r[i], b = r[i + half];
                    r[i] = a * cs[i] - b * sn[i];
                    r[i + half] = b * cs[i] + a * sn[i];
                }
            };
            for (int hh = 0; hh < o->nq; ++hh) rot(&q[size_t(t * qr + hh * hd)]);
            for (int hh = 0; hh < o->nkv; ++hh) {
                rot(&k[size_t(t * kr + hh * hd)]);
                const int64_t blk = d->slot[t] / 16, off = d->slot[t] % 16;
                for (int64_t dd = 0; dd < hd; ++dd) {
                    KC[size_t(((blk * o->nkv + hh) * 16 + off) * hd + dd)] = k[size_t(t * kr + hh * hd + dd)];
                    VC[size_t(((blk * o->nkv + hh) * 16 + off) * hd + dd)] = v[size_t(t * kr + hh * hd + dd)];
                }
            }
        }
        // attention: token t of entry e sees keys [0, pos[t]] through the block table
        const float scale = float(1.0 / std::sqrt(double(hd)));
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
        for (int64_t t = 0; t < T; ++t)
            for (int hq = 0; hq < o->nq; ++hq) {
                const int e = ent[size_t(t)];
                const int kvh = hq / o->G;
                const int nk = d->pos[t] + 1;
                const int32_t* bt = d->block_table + int64_t(e) * d->max_blocks;
                const float* qv = &q[size_t(t * qr + hq * hd)];
                std::vector<float> s(static_cast<size_t>(nk));
                float mx = -INFINITY;
                for (int key = 0; key < nk; ++key) {
                    const float* kv = &KC[size_t(((int64_t(bt[key / 16]) * o->nkv + kvh) * 16 + key % 16) * hd)];
                    float acc = 0.f;
                    for (int64_t dd = 0; dd < hd; ++dd) acc += qv[dd] * kv[dd];
                    s[size_t(key)] = acc * scale;
                    mx = std::max(mx, s[size_t(key)]);
                }
                double den = 0;
                for (int key = 0; key < nk; ++key) {
                    s[size_t(key)] = std::exp(s[size_t(key)] - mx);
                    den += s[size_t(key)];
                }
                float* out = &att[size_t(t * qr + hq * hd)];
                for (int64_t dd = 0; dd < hd; ++dd) out[dd] = 0.f;
                for (int key = 0; key < nk; ++key) {
                    const float* vv = &VC[size_t(((int64_t(bt[key / 16]) * o->nkv + kvh) * 16 + key % 16) * hd)];
                    const float w = float(s[size_t(key)] / den);
                    for (int64_t dd = 0; dd < hd; ++dd) out[dd] += w * vv[dd];
                }
            }
        sgemm_nt(att.data(), W.wo.data(), part.data(), T, h, qr, false);
        allreduce(o, part.data(), T * h);
        for (int64_t i = 0; i < T * h; ++i) x[size_t(i)] += part[size_t(i)];
        rmsnorm_rows(x.data(), W.g_mlp.data(), xn.data(), T, h, eps);
        sgemm_nt(xn.data(), W.wg.data(), g.data(), T, o->ffn, h, false);
        sgemm_nt(xn.data(), W.wu.data(), u.data(), T, o->ffn, h, false);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < T * o->ffn; ++i) {
            const float a = g[size_t(i)];
            g[size_t(i)] = a / (1.f + std::exp(-a)) * u[size_t(i)];
        }
        sgemm_nt(g.data(), W.wd.data(), part.data(), T, h, o->ffn, false);
        allreduce(o, part.data(), T * h);
        for (int64_t i = 0; i < T * h; ++i) x[size_t(i)] += part[size_t(i)];
    }
    if (hidden) std::memcpy(hidden, x.data(), size_t(T * h) * 4);
    if (logits && o->head && d->n_out > 0) {
        std::vector<float> xo(size_t(d->n_out * h)), xr(size_t(d->n_out * h));
        for (int i = 0; i < d->n_out; ++i)
            std::memcpy(&xr[size_t(i * h)], &x[size_t(int64_t(d->out_rows[i]) * h)], size_t(h) * 4);
        rmsnorm_rows(xr.data(), o->g_final.data(), xo.data(), d->n_out, h, eps);
        sgemm_nt(xo.data(), o->lm_head.data(), logits, d->n_out, o->vl, h, false);
    }
    return 0;
}

int32_t orc_weight(orc* o, const char* name, int32_t layer, float* out, int64_t* rows, int64_t* cols) {
    const std::string n(name);
    const std::vector<float>* w = nullptr;
    int64_t r = 0, c = 0;
    const int64_t h = o->h, qr = int64_t(o->nq) * o->hd, kr = int64_t(o->nkv) * o->hd;
    if (n == "embed") { w = &o->embed; r = o->cfg.vocab; c = h; }
    else if (n == "final_norm") { w = &o->g_final; r = 1; c = h; }
    else if (n == "lm_head") { w = &o->lm_head; r = o->vl; c = h; }
    else if (layer >= 0 && layer < o->L) {
        const Layer& W = o->layers[size_t(layer)];
        if (n == "wq") { w = &W.wq; r = qr; c = h; }
        else if (n == "wk") { w = &W.wk; r = kr; c = h; }
        else if (n == "wv") { w = &W.wv; r = kr; c = h; }
        else if (n == "wo") { w = &W.wo; r = h; c = qr; }
        else if (n == "wg") { w = &W.wg; r = o->ffn; c = h; }
        else if (n == "wu") { w = &W.wu; r = o->ffn; c = h; }
        else if (n == "wd") { w = &W.wd; r = h; c = o->ffn; }
        else if (n == "attn_norm") { w = &W.g_attn; r = 1; c = h; }
        else if (n == "mlp_norm") { w = &W.g_mlp; r = 1; c = h; }
    }
    if (!w || w->empty()) return 1;
    if (rows) *rows = r;
    if (cols) *cols = c;
    if (out) std::memcpy(out, w->data(), size_t(r * c) * 4);
    return 0;
}

}  // extern "C"
