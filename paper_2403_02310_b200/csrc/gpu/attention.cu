// K1: mixed-batch paged attention — prefill chunks and decodes in ONE launch.
//
// The launch is driven by a host-built work list over the varlen
// token->request map (cu_q / ctx_len / block tables). For an entry with n
// tokens at prefix p, query token j sits at absolute position p + j and sees
// keys [0, p + j] (its cached prefix plus the causal part of its own chunk);
// a decode is the n = 1 case and sees its whole cache. This is the real
// counterpart of the reference cost model's chunk term q*c^2 + kv*c*prefix and
// decode term a*prefix (reference proj/src/costmodel.cpp:28-37, :48-52).
//
// GQA packing: for KV head h the G = nq/nkv query heads sharing it are packed
// into the MMA row dimension together with the tokens (row = j * G + i), so
// every K/V byte streamed from HBM feeds G query heads.
//
// Item modes (CTA-uniform, 4 warps):
//   row mode  (rows > 16, prefill tiles): warp w owns rows [16w, 16w+16) and
//             walks the whole key range; flash-attention-2 style loop.
//   key mode  (rows <= 16, decodes):      all warps share the rows; each warp
//             takes a 16-key slice of every 64-key tile, and the four partial
//             softmax states are merged in shared memory at the end.
// Long key ranges are split across CTAs (split-KV); partial (m, l, O) go to a
// workspace and attention_combine merges them in a fixed order (deterministic).
//
// K/V pages ([block][kv_head][16][hd], 4 KB contiguous at hd=128) are stored
// pre-swizzled (common.cuh kv_page_elem: per 64-column half, the SWIZZLE_128B
// image of a 16 x 64 box), so 1D bulk copies (cp.async.bulk, 2 KB each) land
// them into a kStages-deep full/empty mbarrier ring exactly as a swizzled
// tensor-map load would — at the 1D engine's higher measured read ceiling
// (profiles/r02/hbm_read_bench.txt) — issued by a dedicated producer warp: no per-thread address math or
// block-table loads in the compute warps, and no CTA-wide barrier per tile.
// S = QK^T and O += PV use mma.sync m16n8k16 (bf16 in, fp32 accumulate); the
// decode path is HBM-bound, so the MMA flavour does not limit it.
#include <cfloat>
#include <climits>

#include "common.cuh"
#include "kernels.cuh"

namespace ssk {

namespace {

constexpr int kWarps = 4;
constexpr int kKeysPerTile = 64;
constexpr int kRowsPerTile = 64;
constexpr int kStages = 3;  // 2 CTAs/SM x 2 tiles in flight = 128 KB of K/V outstanding per SM

constexpr int kTcRows = 128;  // rows of a tensor-core (prefill) item

template <int HD>
struct AttnSmem {
    static constexpr int Q_BYTES = kRowsPerTile * HD * 2;
    static constexpr int KV_TILE = kKeysPerTile * HD * 2;  // [HD/64 halves][64 keys][128 B]
    static constexpr int STAGE = 2 * KV_TILE;              // K + V
    static constexpr int BAR_OFF = Q_BYTES + kStages * STAGE;
    // 256 B of barriers + 704 B of alignment slack (the dynamic window starts 1 KB-aligned
    // in practice; checked at run time) keep two decode CTAs per SM within 228 KB at hd = 128
    static constexpr int TOTAL = BAR_OFF + 256 + 704;
};

// Tensor-core prefill kernel smem: NH halves of 128 rows, each with its Q [HD/64][128
// rows][128 B] and NP P buffers [128 rows][64 keys] bf16, and STAGES K/V stages shared by
// the halves — all SWIZZLE_128B, K-major (V read MN-major).
//   MODE 1 "paired" (NH = 2, NP = 2): one CTA per SM; two row tiles of the same (entry,
//     kv head) share every K/V tile and their softmax warps interleave on the SM (when the
//     256-row items still fill the machine).
//   MODE 3 "deep" (NH = 1, NP = 2): one CTA per SM, 128-row tiles, 5 K/V stages.
//   MODE 2 "compact" (NH = 1, NP = 1): the decode CTA's footprint, so it co-resides with
//     the decode kernel's CTAs and runs beside them.
template <int HD, int MODE>
struct TcCfg {
    using S = AttnSmem<HD>;
    static constexpr int NH = MODE == 1 ? 2 : 1;
    static constexpr int NP = MODE == 2 ? 1 : 2;
    static constexpr int STAGE = S::STAGE;
    static constexpr int QH = kTcRows * HD * 2;           // one half's Q
    static constexpr int P_ONE = kTcRows * kKeysPerTile * 2;
    static constexpr int BUDGET = MODE != 2 ? 232448 - 1024 : 115648;  // compact: half an SM
    static constexpr int STAGES_FIT = (BUDGET - 960 - NH * (QH + NP * P_ONE)) / STAGE;
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
    static constexpr int STAGE0 = NH * QH;
    static constexpr int P = STAGE0 + STAGES * STAGE;     // half h's buffers at P + h * NP * P_ONE
    static constexpr int BAR = P + NH * NP * P_ONE;
    static constexpr int TOTAL = BAR + 256 + 704;
    static constexpr int THREADS = (4 * NH + 2) * 32;     // softmax warps, producer, MMA issuer
    static_assert(STAGES >= 2, "tensor-core attention needs two K/V stages");
};

// Per-half barriers of the tensor-core kernel: S ready [2], PV done [2], P published [2].
struct TcBars {
    uint64_t *sbar, *obar, *pready;
};
// K/V tiles half h needs: through the causal limit of its last row (>= 1 tile if it has rows).
__device__ __forceinline__ int tc_tiles(const AttnParams& p, const AttnItem& it, int h) {
    const int nr = min(max(it.nrows - h * kTcRows, 0), kTcRows);
    if (nr == 0) return 0;
    const int e = it.entry;
    const int prefix = p.ctx_len[e] - (p.cu_q[e + 1] - p.cu_q[e]);
    const int kneed = min(prefix + (it.row0 + h * kTcRows + nr - 1) / p.group + 1, it.key1);
    return max(1, (kneed - it.key0 + kKeysPerTile - 1) / kKeysPerTile);
}

// Q tile: rows of HD*2 bytes, 16-byte chunks XOR-swizzled by row.
template <int HD>
__device__ __forceinline__ uint32_t swz_q(int row, int c) {
    return uint32_t(row * (HD * 2) + ((c ^ (row & 7)) << 4));
}
// K/V tile in shared memory (SWIZZLE_128B image): [c / 8 half][key][128 B].
__device__ __forceinline__ uint32_t swz_kv(int key, int c) {
    return uint32_t((c >> 3) * (kKeysPerTile * 128) + key * 128 + (((c & 7) ^ (key & 7)) << 4));
}

// KPW = keys handled per warp per 64-key tile (64: row mode, 16: key mode).
template <int HD, int KPW>
__device__ __forceinline__ void attend(const AttnParams& p,
                                       const AttnItem& it, uint8_t* smem, int qrow_base, int kofs,
                                       float (&O)[HD / 8][4], float (&m)[2], float (&l)[2]) {
    using S = AttnSmem<HD>;
    constexpr int NT = KPW / 8;  // n8 tiles of S per warp
    const int lane = threadIdx.x & 31;
    uint8_t* sQ = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
    const int e = it.entry;
    const int tok0 = p.cu_q[e];
    const int ntok = p.cu_q[e + 1] - tok0;
    const int prefix = p.ctx_len[e] - ntok;

    // Q fragments for this warp's 16 rows, all HD/16 k-steps.
    uint32_t qa[HD / 16][4];
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
        const int r = qrow_base + (lane & 15);
        ldsm_x4(smem_u32(sQ) + swz_q<HD>(r, ks * 2 + (lane >> 4)), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    }
    // causal limits of the two rows this thread holds (unused rows see everything:
    // their Q is zero, so they stay finite and are never stored)
    int lim[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int r = qrow_base + (lane >> 2) + hr * 8;
        lim[hr] = r < it.nrows ? prefix + (it.row0 + r) / p.group : INT_MAX;
    }
    const int lim_lo = __reduce_min_sync(0xffffffffu, min(lim[0], lim[1]));
    m[0] = m[1] = -INFINITY;
    l[0] = l[1] = 0.f;
#pragma unroll
    for (int dt = 0; dt < HD / 8; ++dt) O[dt][0] = O[dt][1] = O[dt][2] = O[dt][3] = 0.f;

    uint64_t* empty = full + 8;  // barrier block layout: see attention_kernel
    const int ntiles = (it.key1 - it.key0 + kKeysPerTile - 1) / kKeysPerTile;
    for (int t = 0; t < ntiles; ++t) {
        const int kbase = it.key0 + t * kKeysPerTile;
        const int st = t % kStages;
        uint8_t* sK = smem + S::Q_BYTES + st * S::STAGE;
        uint8_t* sV = sK + S::KV_TILE;
        mbar_wait(&full[st], uint32_t((t / kStages) & 1));
#if defined(SS_ATTN_EXP) && SS_ATTN_EXP == 1  // dev experiment: consumers release stages unread
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        continue;
#endif

        // S = Q K^T for this warp's key slice
        float s[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
#pragma unroll
            for (int nt = 0; nt < NT; nt += 2) {
                const int key = kofs + nt * 8 + ((lane >> 4) << 3) + (lane & 7);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(smem_u32(sK) + swz_kv(key, ks * 2 + ((lane >> 3) & 1)), b0, b1, b2, b3);
                mma_bf16_16816(s[nt], qa[ks], b0, b1);
                mma_bf16_16816(s[nt + 1], qa[ks], b2, b3);
            }
        }
        // mask only where a row's causal limit or the range end cuts this slice
        const int klast = kbase + kofs + KPW - 1;
        if (klast > lim_lo || klast >= it.key1) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int key = kbase + kofs + nt * 8 + 2 * (lane & 3) + (c & 1);
                    if (key > lim[c >> 1] || key >= it.key1) s[nt][c] = -INFINITY;
                }
        }
        float mt[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            mt[0] = fmaxf(mt[0], fmaxf(s[nt][0], s[nt][1]));
            mt[1] = fmaxf(mt[1], fmaxf(s[nt][2], s[nt][3]));
        }
        float alpha[2], msub[2];
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            mt[hr] = fmaxf(mt[hr], __shfl_xor_sync(0xffffffffu, mt[hr], 1));
            mt[hr] = fmaxf(mt[hr], __shfl_xor_sync(0xffffffffu, mt[hr], 2));
            const float mn = fmaxf(m[hr], mt[hr] * p.scale_log2);
            msub[hr] = mn == -INFINITY ? 0.f : mn;
            alpha[hr] = exp2f(m[hr] - msub[hr]);
            m[hr] = mn;
            l[hr] *= alpha[hr];
        }
        if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
            for (int dt = 0; dt < HD / 8; ++dt) {
                O[dt][0] *= alpha[0];
                O[dt][1] *= alpha[0];
                O[dt][2] *= alpha[1];
                O[dt][3] *= alpha[1];
            }
        }
        uint32_t pa[NT / 2][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const float p0 = exp2f(fmaf(s[nt][0], p.scale_log2, -msub[0]));
            const float p1 = exp2f(fmaf(s[nt][1], p.scale_log2, -msub[0]));
            const float p2 = exp2f(fmaf(s[nt][2], p.scale_log2, -msub[1]));
            const float p3 = exp2f(fmaf(s[nt][3], p.scale_log2, -msub[1]));
            l[0] += p0 + p1;
            l[1] += p2 + p3;
            pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
            pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
        }
        // O += P V
#pragma unroll
        for (int kk = 0; kk < NT / 2; ++kk) {
            const uint32_t a[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
            const int key = kofs + kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
            for (int dt = 0; dt < HD / 8; dt += 2) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(smem_u32(sV) + swz_kv(key, dt + (lane >> 4)), b0, b1, b2, b3);
                mma_bf16_16816(O[dt], a, b0, b1);
                mma_bf16_16816(O[dt + 1], a, b2, b3);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with stage st
    }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        l[hr] += __shfl_xor_sync(0xffffffffu, l[hr], 1);
        l[hr] += __shfl_xor_sync(0xffffffffu, l[hr], 2);
    }
}

// Merges the partial (m, l, O) of every split of a group into the final bf16
// output, in split order (deterministic). Run by the CTA that finishes a
// group's last split; 128 compute threads.
template <int HD>
__device__ __forceinline__ void combine_group(const AttnParams& p, const AttnCombine& c, int tid) {
    for (int idx = tid; idx < c.nrows * HD; idx += kWarps * 32) {
        const int r = idx / HD, d = idx % HD;
        float M = -INFINITY;
        for (int s = 0; s < c.nsplit; ++s) M = fmaxf(M, __ldcg(p.part_ml + size_t(c.part + s * c.stride + r) * 2));
        const float Ms = M == -INFINITY ? 0.f : M;
        float L = 0.f, o = 0.f;
        for (int s = 0; s < c.nsplit; ++s) {
            const size_t slot = size_t(c.part + s * c.stride + r);
            const float f = exp2f(__ldcg(p.part_ml + slot * 2) - Ms);
            L += __ldcg(p.part_ml + slot * 2 + 1) * f;
            o += __ldcg(p.part_o + slot * HD + d) * f;
        }
        const int gr = c.row0 + r;
        const int tok = p.cu_q[c.entry] + gr / p.group;
        const int hq = c.kv_head * p.group + gr % p.group;
        p.o[(size_t(tok) * p.nq_l + hq) * HD + d] = __float2bfloat16(L > 0.f ? o / L : 0.f);
    }
}

// After a split's partials are written: the last split of the group to finish
// (threadFenceReduction pattern) merges all splits and resets the counter.
template <int HD>
__device__ __forceinline__ void finish_split(const AttnParams& p, const AttnItem& it, int* s_flag) {
    if (it.comb < 0) return;
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");
    if (threadIdx.x == 0) {
        const AttnCombine c = p.combines[it.comb];
        *s_flag = atomicAdd(&p.comb_count[it.comb], 1) == c.nsplit - 1;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");
    if (!*s_flag) return;
    __threadfence();
    combine_group<HD>(p, p.combines[it.comb], threadIdx.x);
    if (threadIdx.x == 0) p.comb_count[it.comb] = 0;
}

// Writes one row's final (normalised bf16) or partial (fp32 O, m, l) result.
template <int HD>
__device__ __forceinline__ void emit_pair(const AttnParams& p, const AttnItem& it, int r, int d, float o0, float o1,
                                          float mm, float ll) {
    if (r >= it.nrows) return;
    const int gr = it.row0 + r;
    if (it.part < 0) {
        const int tok = p.cu_q[it.entry] + gr / p.group;
        const int hq = it.kv_head * p.group + gr % p.group;
        const float inv = ll > 0.f ? 1.f / ll : 0.f;
        *reinterpret_cast<uint32_t*>(p.o + (size_t(tok) * p.nq_l + hq) * HD + d) = pack_bf16(o0 * inv, o1 * inv);
    } else {
        *reinterpret_cast<float2*>(p.part_o + size_t(it.part + r) * HD + d) = make_float2(o0, o1);
        if (d == 0) *reinterpret_cast<float2*>(p.part_ml + size_t(it.part + r) * 2) = make_float2(mm, ll);
    }
}


// ---- tensor-core prefill tile (tcgen05): 128 GQA-packed rows x 64-key tiles.
// Warp 0 (one elected lane) issues S = Q K^T into a TMEM double buffer and O += P V
// into a TMEM accumulator; each of the 4 warps' threads owns one row (TMEM lane), so
// the online softmax is thread-local: no shuffles. The running max is refreshed only
// when it grows by more than 2^8 (log2 units), which keeps rescales of the O row in
// TMEM rare while every p = 2^(s - m) stays <= 256 (exact in fp32, relative in bf16).
__device__ __forceinline__ void tmem_st32_attn(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ float ex2_approx(float x) {  // 2^x, -inf -> 0
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ bool elect_lane() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}
// MN-major SWIZZLE_128B operand (V as B of O += P V: N = head dim contiguous, K = keys):
// 8-key groups 1 KB apart (SBO), 64-column halves of the head dim LBO apart.
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo) {
    return (uint64_t((smem_addr >> 4) & 0x3FFFu)) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
           (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// Warp roles of the tensor-core kernel: warps 0-3 softmax (thread = row = TMEM
// lane), warp 4 TMA producer, warp 5 MMA issuer. Per 64-key tile t the issuer runs
// S(t) = Q K(t)^T into TMEM buffer t & 1 and, once the softmax warps have published
// P(t - 1) (mbarrier, one arrival per warp), O += P(t - 1) V(t - 1); P is double
// buffered in smem, so softmax(t) overlaps PV(t - 1) and S(t + 1).
template <int HD, int MODE>
__device__ __forceinline__ void mma_warp_tc(const AttnParams& p, const AttnItem& it, uint8_t* smem, uint64_t* full,
                                            uint64_t* empty, const TcBars (&bars)[2], uint32_t tbase) {
    using S = AttnSmem<HD>;
    using C = TcCfg<HD, MODE>;
    constexpr int NST = C::STAGES, NH = C::NH, NP = C::NP;
    int nth[2] = {tc_tiles(p, it, 0), NH > 1 ? tc_tiles(p, it, 1) : 0};
    const int nt = max(nth[0], nth[1]);
    constexpr uint32_t idS = umma_idesc_bf16(kTcRows, kKeysPerTile);
    constexpr uint32_t idO = umma_idesc_bf16(kTcRows, HD) | (1u << 16);  // B (V) MN-major
    const uint32_t qa = smem_u32(smem), sa = smem_u32(smem + C::STAGE0), pa = smem_u32(smem + C::P);
    for (int t = 0; t <= nt; ++t) {
        if (t < nt) {  // S_h(t) = Q_h K(t)^T into half h's TMEM buffer t & 1
            // (S buffer t & 1 was last read by softmax(t - 2): P(t - 2) was awaited before PV(t - 2))
            const int st = t % NST;
            mbar_wait(&full[st], uint32_t((t / NST) & 1));
            tc_fence_after();
            if (elect_lane()) {
                const uint32_t ka = sa + st * S::STAGE;
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    if (t >= nth[h]) continue;
#pragma unroll
                    for (int ks = 0; ks < HD / 16; ++ks) {
                        const int hh = ks >> 2, kk = ks & 3;
                        umma_bf16(tbase + uint32_t(h * 256 + (t & 1) * 64),
                                  umma_desc_sw128(qa + h * C::QH + hh * kTcRows * 128) + uint64_t(2 * kk),
                                  umma_desc_sw128(ka + hh * kKeysPerTile * 128) + uint64_t(2 * kk), idS, ks > 0 ? 1u : 0u);
                    }
                    umma_commit(&bars[h].sbar[t & 1]);
                }
            }
            __syncwarp();
        }
        if (t >= 1) {  // O_h += P_h(u) V(u), u = t - 1, once half h published P_h(u)
            const int u = t - 1;
            const uint32_t va = sa + (u % NST) * S::STAGE + S::KV_TILE;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                if (u >= nth[h]) continue;
                mbar_wait(&bars[h].pready[u & 1], uint32_t((u >> 1) & 1));
                tc_fence_after();
                if (elect_lane()) {
                    const uint32_t pb = pa + (h * NP + u % NP) * C::P_ONE;
#pragma unroll
                    for (int kk = 0; kk < kKeysPerTile / 16; ++kk)
                        umma_bf16(tbase + uint32_t(h * 256 + 128), umma_desc_sw128(pb) + uint64_t(2 * kk),
                                  umma_desc_sw128_mn(va + kk * 16 * 128, kKeysPerTile * 128), idO,
                                  (u > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&bars[h].obar[u & 1]);
                }
                __syncwarp();
            }
            if (elect_lane()) umma_commit(&empty[u % NST]);  // K/V stage free once S(u), PV(u) retire
            __syncwarp();
        }
    }
}

template <int HD, int MODE>
__device__ __forceinline__ void softmax_warps_tc(const AttnParams& p, const AttnItem& it, uint8_t* smem,
                                                 const TcBars (&bars)[2], uint32_t tbase0, int warp, int lane) {
    using C = TcCfg<HD, MODE>;
    constexpr int NP = C::NP;
    const int h = warp >> 2, wq = warp & 3;  // half of the item, TMEM lane quarter
    const int nt = tc_tiles(p, it, h);
    if (nt == 0) return;  // this half has no rows
    // (the halves' barriers are contiguous, 6 per half: no dynamic indexing of `bars`)
    uint64_t* sbar = bars[0].sbar + 6 * h;
    uint64_t* obar = bars[0].obar + 6 * h;
    uint64_t* pready = bars[0].pready + 6 * h;
    const uint32_t tbase = tbase0 + uint32_t(h * 256);
    const int r = h * kTcRows + wq * 32 + lane;  // row of the item
    const int rl = wq * 32 + lane;               // row of the half == TMEM lane
    const int e = it.entry;
    const int tok0 = p.cu_q[e];
    const int ntok = p.cu_q[e + 1] - tok0;
    const int prefix = p.ctx_len[e] - ntok;
    const int lim = r < it.nrows ? prefix + (it.row0 + r) / p.group : -1;  // last visible key
    const uint32_t lane_base = uint32_t(wq * 32) << 16;
    const uint32_t tO = tbase + 128;
    float m = -INFINITY, l = 0.f;
    for (int t = 0; t < nt; ++t) {
        mbar_wait(&sbar[t & 1], uint32_t((t >> 1) & 1));
        tc_fence_after();
        uint32_t sv[64];
        tmem_ld32(tbase + lane_base + uint32_t((t & 1) * 64), *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
        tmem_ld32(tbase + lane_base + uint32_t((t & 1) * 64 + 32), *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
        tmem_wait_ld();
        const int kb = it.key0 + t * kKeysPerTile;
        const int kend = min(lim + 1, it.key1) - kb;  // keys [kb, kb + kend) are visible to this row
        // raw-score max (the scale is positive); the mask pass runs only where a row's
        // causal limit or the range end cuts this tile
        if (__any_sync(0xffffffffu, kend < 64)) {
#pragma unroll
            for (int j = 0; j < 64; ++j)
                if (j >= kend) sv[j] = __float_as_uint(-INFINITY);
        }
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
            mx0 = fmaxf(mx0, __uint_as_float(sv[j]));
            mx1 = fmaxf(mx1, __uint_as_float(sv[j + 1]));
        }
        const float mx = fmaxf(mx0, mx1) * p.scale_log2;
        // lazy max: refresh only on first sight or growth by > 2^8
        float alpha = 1.f;
        if (mx > m + 8.f) {
            alpha = m == -INFINITY ? 1.f : ex2_approx(m - mx);
            m = mx;
        }
        const float msub = m == -INFINITY ? 0.f : m;
        float ls0 = 0.f, ls1 = 0.f;
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const float p0 = ex2_approx(fmaf(__uint_as_float(sv[2 * j]), p.scale_log2, -msub));
            const float p1 = ex2_approx(fmaf(__uint_as_float(sv[2 * j + 1]), p.scale_log2, -msub));
            ls0 += p0;
            ls1 += p1;
            pk[j] = pack_bf16(p0, p1);
        }
        l = l * alpha + (ls0 + ls1);
        // P buffer t % NP was read by PV(t - NP); a rescale of O needs PV(t - 1) retired
        if (t >= NP) {
            mbar_wait(&obar[(t - NP) & 1], uint32_t(((t - NP) >> 1) & 1));
            tc_fence_after();
        }
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
            mbar_wait(&obar[(t - 1) & 1], uint32_t(((t - 1) >> 1) & 1));
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < HD / 32; ++c) {
                uint32_t ov[32];
                tmem_ld32(tO + lane_base + uint32_t(c * 32), ov);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * alpha);
                tmem_st32_attn(tO + lane_base + uint32_t(c * 32), ov);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        // P row -> smem (K-major SWIZZLE_128B: 16-byte chunk j of row r at j ^ (r & 7))
        uint4* prow = reinterpret_cast<uint4*>(smem + C::P + (h * NP + t % NP) * C::P_ONE + rl * 128);
#pragma unroll
        for (int j = 0; j < 8; ++j) prow[j ^ (rl & 7)] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pready[t & 1]);  // one arrival per softmax warp
    }
    // the last PV retires -> O row / l -> bf16 (final) or the unnormalised partial
    mbar_wait(&obar[(nt - 1) & 1], uint32_t(((nt - 1) >> 1) & 1));
    tc_fence_after();
    const bool live = r < it.nrows;
    const int gr = it.row0 + r;
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int c = 0; c < HD / 32; ++c) {
        uint32_t ov[32];
        tmem_ld32(tO + lane_base + uint32_t(c * 32), ov);
        tmem_wait_ld();
        if (!live) continue;
        if (it.part < 0) {
            __nv_bfloat16* dst = p.o + (size_t(tok0 + gr / p.group) * p.nq_l + it.kv_head * p.group + gr % p.group) * HD + c * 32;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                reinterpret_cast<uint4*>(dst)[j] = make_uint4(
                    pack_bf16(__uint_as_float(ov[8 * j + 0]) * inv, __uint_as_float(ov[8 * j + 1]) * inv),
                    pack_bf16(__uint_as_float(ov[8 * j + 2]) * inv, __uint_as_float(ov[8 * j + 3]) * inv),
                    pack_bf16(__uint_as_float(ov[8 * j + 4]) * inv, __uint_as_float(ov[8 * j + 5]) * inv),
                    pack_bf16(__uint_as_float(ov[8 * j + 6]) * inv, __uint_as_float(ov[8 * j + 7]) * inv));
        } else {
            float4* dst = reinterpret_cast<float4*>(p.part_o + size_t(it.part + r) * HD + c * 32);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                dst[j] = make_float4(__uint_as_float(ov[4 * j]), __uint_as_float(ov[4 * j + 1]),
                                     __uint_as_float(ov[4 * j + 2]), __uint_as_float(ov[4 * j + 3]));
            if (c == 0) *reinterpret_cast<float2*>(p.part_ml + size_t(it.part + r) * 2) = make_float2(m, l);
        }
    }
}

// MODE 0: decode / mma.sync items; 1: tensor-core prefill, deep; 2: tensor-core prefill, compact.
template <int HD, int MODE>
__global__ void __launch_bounds__(MODE > 0 ? TcCfg<HD, MODE>::THREADS : (kWarps + 1) * 32) attention_kernel(const AttnParams p) {
    using S = AttnSmem<HD>;
    constexpr bool TC = MODE > 0;
    using C = TcCfg<HD, MODE == 0 ? 2 : MODE>;
    constexpr int NH = TC ? C::NH : 1;
    constexpr int kProd = TC ? 4 * NH : kWarps;  // producer warp; the tc MMA warp follows it
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
    if (pad > 704u) __trap();  // SWIZZLE_128B tiles need 1 KB alignment
    uint8_t* smem = smem_raw + pad;
    const AttnItem it = p.items[blockIdx.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool key_mode = !TC && it.nrows <= 16;
    constexpr bool tc = TC;  // prefill row tile on the tensor cores
    // barrier block (256 B): full[8] empty[8] | split flag | per half {S-ready[2] PV-done[2]
    // P-ready[2]} | TMEM slot
    constexpr int kMaxSt = 8;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (TC ? C::BAR : S::BAR_OFF));
    uint64_t* empty = full + kMaxSt;
    int* split_flag = reinterpret_cast<int*>(full + 2 * kMaxSt);
    uint64_t* hb = full + 2 * kMaxSt + 1;
    const TcBars bars[2] = {{hb, hb + 2, hb + 4}, {hb + 6, hb + 8, hb + 10}};
    uint32_t* tslot = reinterpret_cast<uint32_t*>(hb + 12);
    const int nst = tc ? C::STAGES : kStages;
    const int st0 = tc ? C::STAGE0 : S::Q_BYTES;

    // (mma.sync path: the producer warp initialises the barriers, so it can issue before the
    // CTA-wide barrier below; the other warps touch them only after it)
    if (threadIdx.x == (TC ? 0 : kProd * 32)) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], tc ? 1 : kWarps);  // tc: released by a tcgen05.commit
        }
        for (int i = 0; i < 12; ++i) mbar_init(&hb[i], (i % 6) >= 4 ? 4 : 1);  // P-ready: 4 softmax warps
        mbar_fence_init();
    }
    if constexpr (TC) {  // per half: S double buffer (2 x 64 cols) + O (HD cols)
        if (warp == 0) {
            if constexpr (NH == 2) tmem_alloc<512>(tslot);
            else tmem_alloc<256>(tslot);
        }
    }
    // ---- K/V producer state (warp kProd). Block ids come 32 pages (8 tiles) at a time from
    // one coalesced warp load, fetched a batch ahead, and reach the issuing lane by shuffle:
    // no dependent global load sits between two tiles' issues.
    int pr_ntiles = 0, pr_nvalid = 0, pr_t = 0;
    int32_t pr_cur = 0, pr_nxt = 0;
    uint64_t pr_pol = 0;
    const int32_t* pr_bt = p.block_table + size_t(it.entry) * p.max_blocks;
    const int pr_pg0 = it.key0 >> 4;  // key0 is a multiple of 64
    auto pr_batch = [&](int b) {
        const int lb = pr_pg0 + 32 * b + lane;
        return __ldg(pr_bt + (lb < pr_nvalid ? lb : 0));  // pages past the context: a valid page, masked
    };
    auto pr_issue = [&](int t) {
        if (t > 0 && (t & 7) == 0) {
            pr_cur = pr_nxt;
            if (t + 8 < pr_ntiles) pr_nxt = pr_batch((t >> 3) + 1);
        }
        int32_t blk[4];
#pragma unroll
        for (int pg = 0; pg < 4; ++pg) blk[pg] = __shfl_sync(0xffffffffu, pr_cur, ((t & 7) << 2) + pg);
        const int st = t % nst;
        // one 2 KB copy per lane: a tile's 4 pages x HD/64 halves x {K, V} issue in parallel
        // (a single issuing thread serialises them: measured 1.5x slower)
        constexpr int kOps = 4 * (HD / 64) * 2;
        if (t >= nst) mbar_wait(&empty[st], uint32_t(((t / nst) - 1) & 1));
        if (lane < kOps) {
            if (lane == 0) mbar_arrive_expect_tx(&full[st], 2 * S::KV_TILE);
            const int kv = lane & 1, hh = (lane >> 1) % (HD / 64), pg = lane / (2 * (HD / 64));
            // the half-page is stored pre-swizzled (kv_page_elem): one 2 KB bulk copy lands
            // the same shared-memory image a SWIZZLE_128B 16 x 64 tensor box would
            const __nv_bfloat16* src =
                (kv ? p.vc : p.kc) + (int64_t(blk[pg]) * p.nkv_l + it.kv_head) * (16 * HD) + hh * (16 * 64);
            uint8_t* dst = smem + st0 + st * S::STAGE + kv * S::KV_TILE + hh * (kKeysPerTile * 128) + pg * 16 * 128;
            bulk_load_hint(dst, src, 16 * 128, &full[st], pr_pol);
        }
        __syncwarp();
    };
    if (warp == kProd) {
        // the item list, block tables and lengths were uploaded before the forward's first kernel
        pr_ntiles = TC ? max(tc_tiles(p, it, 0), NH > 1 ? tc_tiles(p, it, 1) : 0)
                       : (it.key1 - it.key0 + kKeysPerTile - 1) / kKeysPerTile;
        pr_nvalid = (p.ctx_len[it.entry] + 15) >> 4;
        pr_cur = pr_batch(0);
        pr_nxt = pr_ntiles > 8 ? pr_batch(1) : 0;
        // a decode's K/V streams through once: first out of L2, so the chunk's freshly
        // appended K/V and the next projection's operands stay resident
        pr_pol = it.nrows <= 16 ? ((p.kv_hint & 1) ? l2_policy_evict_first() : l2_policy_evict_normal())
                                : ((p.kv_hint & 2) ? l2_policy_evict_last() : l2_policy_evict_normal());
        if constexpr (!TC) {
            if (!p.wait_at_end) {
                // Tiles of cached keys only (positions before this step's tokens) do not depend on
                // the preceding kernels: the forward's first kernel passes its grid-dependency
                // wait before it lets any later kernel start, so every earlier step's K/V writes
                // are complete. Up to a ring's worth is in flight before this CTA's wait — while
                // PDL keeps it resident beside the QKV GEMM's tail.
                __syncwarp();  // barrier init (lane 0) before any lane issues
                const int ntok = p.cu_q[it.entry + 1] - p.cu_q[it.entry];
                const int cached = (p.ctx_len[it.entry] - ntok - it.key0) / kKeysPerTile;
                const int npre = min(min(cached, nst), pr_ntiles);
                for (; pr_t < npre; ++pr_t) pr_issue(pr_t);
            }
        }
    }
    // Grid dependencies (see attention_launch): the first of the two attention launches
    // waits for the QKV kernel and triggers its dependent only after that wait; the second
    // skips the start wait (its CTAs exist only once every CTA of the first has waited) and
    // waits at its end, so its completion covers both.
    if (p.wait_at_end) {
        pdl_launch_dependents();
    } else {
        if (key_mode && p.kv_pf_pages > 0) {
            // The cached pages of this decode item do not depend on the preceding kernels
            // (only the last page receives this step's K/V, from the QKV epilogue): CTAs that
            // PDL makes resident while the QKV GEMM still runs (on the SMs its tiles leave
            // idle) ask L2 for the first pages, using HBM the GEMM leaves idle. The block
            // table and items were uploaded before the forward's first kernel.
            const int32_t* bt = p.block_table + size_t(it.entry) * p.max_blocks;
            const int pg0 = it.key0 >> 4;
            const int npg = min(p.kv_pf_pages, ((it.key1 - 1) >> 4) - pg0);
            const uint32_t page_bytes = uint32_t(p.block_size) * HD * 2;
            for (int i = threadIdx.x; i < 2 * npg; i += blockDim.x) {
                const int32_t blk = __ldg(bt + pg0 + (i >> 1));
                const __nv_bfloat16* src =
                    ((i & 1) ? p.vc : p.kc) + (size_t(blk) * p.nkv_l + it.kv_head) * size_t(p.block_size) * HD;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(page_bytes) : "memory");
            }
        }
        pdl_wait();  // q / KV of this layer come from the preceding kernels
        pdl_launch_dependents();
    }
    // stage the Q tile (rows beyond nrows are zero)
    {
        constexpr int CH = HD / 8;
        const int e = it.entry, tok0 = p.cu_q[e];
        const int nr = key_mode ? 16 : (tc ? NH * kTcRows : kRowsPerTile);
        for (int idx = threadIdx.x; idx < nr * CH; idx += blockDim.x) {
            const int r = idx / CH, c = idx % CH;
            // tc: per half, UMMA K-major SWIZZLE_128B image [c / 8][row][128 B]
            const int rh = r & (kTcRows - 1);
            const uint32_t so = smem_u32(smem) + (tc ? uint32_t((r / kTcRows) * C::QH + (c >> 3) * (kTcRows * 128) + rh * 128 +
                                                                (((c & 7) ^ (rh & 7)) << 4))
                                                   : swz_q<HD>(r, c));
            if (r < it.nrows) {
                const int gr = it.row0 + r;
                const __nv_bfloat16* src =
                    p.q + (size_t(tok0 + gr / p.group) * p.nq_l + it.kv_head * p.group + gr % p.group) * HD + c * 8;
                cp_async16(so, src);
            } else {
                cp_async_zero16(so, p.q);
            }
        }
        cp_async_commit();
        cp_async_wait<0>();
        if constexpr (TC) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // Q is read by tcgen05.mma
            tc_fence_before();
            __syncthreads();
            tc_fence_after();
        } else {
            __syncthreads();
        }
    }

    if (warp == kProd) {  // ---- producer warp: K/V half-pages by bulk copy into the ring
        for (int t = pr_t; t < pr_ntiles; ++t) pr_issue(t);
        if (p.wait_at_end) pdl_wait();
        return;
    }

    if constexpr (TC) {
        if (warp == kProd + 1) {
            mma_warp_tc<HD, MODE>(p, it, smem, full, empty, bars, *tslot);
            return;
        }
        softmax_warps_tc<HD, MODE>(p, it, smem, bars, *tslot, warp, lane);
        if (p.wait_at_end) pdl_wait();
        if (NH == 1 && p.fused_combine) finish_split<HD>(p, it, split_flag);
        tc_fence_before();
        asm volatile("bar.sync 1, %0;" ::"n"(NH * kWarps * 32) : "memory");
        if (warp == 0) {
            tc_fence_after();
            if constexpr (NH == 2) tmem_dealloc<512>(*tslot);
            else tmem_dealloc<256>(*tslot);
        }
        return;
    } else {
    float O[HD / 8][4], m[2], l[2];
    if (!key_mode) {
        attend<HD, 64>(p, it, smem, warp * 16, 0, O, m, l);
        const int r0 = warp * 16 + (lane >> 2);
#pragma unroll
        for (int dt = 0; dt < HD / 8; ++dt) {
            const int d = dt * 8 + 2 * (lane & 3);
            emit_pair<HD>(p, it, r0, d, O[dt][0], O[dt][1], m[0], l[0]);
            emit_pair<HD>(p, it, r0 + 8, d, O[dt][2], O[dt][3], m[1], l[1]);
        }
        if (p.fused_combine) finish_split<HD>(p, it, split_flag);
        if (p.wait_at_end) pdl_wait();
        return;
    }

    attend<HD, 16>(p, it, smem, 0, warp * 16, O, m, l);
    // merge the four warps' partial softmax states (K/V stages reused as scratch,
    // once every compute warp is past its last tile)
    asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");
    float* sO = reinterpret_cast<float*>(smem + S::Q_BYTES);  // [4][16][HD]
    float* sML = sO + kWarps * 16 * HD;                        // [4][16][2]
    {
        const int r0 = lane >> 2;
#pragma unroll
        for (int dt = 0; dt < HD / 8; ++dt) {
            const int d = dt * 8 + 2 * (lane & 3);
            *reinterpret_cast<float2*>(&sO[(warp * 16 + r0) * HD + d]) = make_float2(O[dt][0], O[dt][1]);
            *reinterpret_cast<float2*>(&sO[(warp * 16 + r0 + 8) * HD + d]) = make_float2(O[dt][2], O[dt][3]);
        }
        if ((lane & 3) == 0) {
            sML[(warp * 16 + r0) * 2] = m[0];
            sML[(warp * 16 + r0) * 2 + 1] = l[0];
            sML[(warp * 16 + r0 + 8) * 2] = m[1];
            sML[(warp * 16 + r0 + 8) * 2 + 1] = l[1];
        }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");
    for (int idx = threadIdx.x; idx < it.nrows * (HD / 2); idx += kWarps * 32) {
        const int r = idx / (HD / 2), d = (idx % (HD / 2)) * 2;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sML[(w * 16 + r) * 2]);
        const float Ms = M == -INFINITY ? 0.f : M;
        float L = 0.f, o0 = 0.f, o1 = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float f = exp2f(sML[(w * 16 + r) * 2] - Ms);
            L += sML[(w * 16 + r) * 2 + 1] * f;
            const float2 ov = *reinterpret_cast<const float2*>(&sO[(w * 16 + r) * HD + d]);
            o0 += ov.x * f;
            o1 += ov.y * f;
        }
        emit_pair<HD>(p, it, r, d, o0, o1, M, L);
    }
    if (p.fused_combine) finish_split<HD>(p, it, split_flag);
    if (p.wait_at_end) pdl_wait();
    }
}

template <int HD>
__global__ void attention_combine_kernel(const AttnParams p) {
    pdl_launch_dependents();
    pdl_wait();
    const AttnCombine c = p.combines[blockIdx.x];
    for (int idx = threadIdx.x; idx < c.nrows * HD; idx += blockDim.x) {
        const int r = idx / HD, d = idx % HD;
        float M = -INFINITY;
        for (int s = 0; s < c.nsplit; ++s) M = fmaxf(M, p.part_ml[size_t(c.part + s * c.stride + r) * 2]);
        const float Ms = M == -INFINITY ? 0.f : M;
        float L = 0.f, o = 0.f;
        for (int s = 0; s < c.nsplit; ++s) {
            const size_t slot = size_t(c.part + s * c.stride + r);
            const float f = exp2f(p.part_ml[slot * 2] - Ms);
            L += p.part_ml[slot * 2 + 1] * f;
            o += p.part_o[slot * HD + d] * f;
        }
        const int gr = c.row0 + r;
        const int tok = p.cu_q[c.entry] + gr / p.group;
        const int hq = c.kv_head * p.group + gr % p.group;
        p.o[(size_t(tok) * p.nq_l + hq) * HD + d] = __float2bfloat16(L > 0.f ? o / L : 0.f);
    }
}

template <int HD>
cudaError_t launch_hd(const AttnParams& p, cudaStream_t st) {
    static bool attr[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(attention_kernel<HD, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             TcCfg<HD, 1>::TOTAL);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(attention_kernel<HD, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     TcCfg<HD, 2>::TOTAL);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(attention_kernel<HD, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     TcCfg<HD, 3>::TOTAL);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(attention_kernel<HD, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     AttnSmem<HD>::TOTAL);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    // items[0, n_tc): tensor-core prefill tiles; the rest: decode / mma.sync items
    const int n_tc = p.tc ? p.n_tc : 0, n_rest = p.n_items - n_tc;
    AttnParams pt = p, pd = p;
    pd.items = p.items + n_tc;
    const dim3 bd((kWarps + 1) * 32);
    if (n_tc > 0 && p.tc == 2 && p.tc2_first > 0 && n_rest > 0) {  // dev: compact prefill CTAs first, decodes beside them
        pt.wait_at_end = 0;
        pd.wait_at_end = 1;
        cudaError_t e = launch_pdl(attention_kernel<HD, 2>, dim3(n_tc), dim3(TcCfg<HD, 2>::THREADS), TcCfg<HD, 2>::TOTAL,
                                   st, 1, pt);
        if (e != cudaSuccess || n_rest == 0) return e;
        return launch_pdl(attention_kernel<HD, 0>, dim3(n_rest), bd, AttnSmem<HD>::TOTAL, st, 1, pd);
    }
    if (n_tc > 0 && p.tc == 2 && n_rest > 0) {
        // enough HBM-streaming decode CTAs to fill the machine: they go first, and the
        // compact prefill CTAs run beside them (in the SMs' remaining shared memory)
        pd.wait_at_end = 0;
        pt.wait_at_end = 1;
        cudaError_t e = launch_pdl(attention_kernel<HD, 0>, dim3(n_rest), bd, AttnSmem<HD>::TOTAL, st, 1, pd);
        if (e != cudaSuccess) return e;
        return launch_pdl(attention_kernel<HD, 2>, dim3(n_tc), dim3(TcCfg<HD, 2>::THREADS), TcCfg<HD, 2>::TOTAL, st, 1,
                          pt);
    }
    if (n_tc > 0) {  // prefill-heavy: the deep prefill kernel first, the decodes beside / after it
        pt.wait_at_end = 0;
        cudaError_t e =
            p.tc == 1 ? launch_pdl(attention_kernel<HD, 1>, dim3(n_tc), dim3(TcCfg<HD, 1>::THREADS), TcCfg<HD, 1>::TOTAL,
                                   st, 1, pt)
                      : launch_pdl(attention_kernel<HD, 3>, dim3(n_tc), dim3(TcCfg<HD, 3>::THREADS), TcCfg<HD, 3>::TOTAL,
                                   st, 1, pt);
        if (e != cudaSuccess || n_rest == 0) return e;
        pd.wait_at_end = 1;
    } else {
        pd.wait_at_end = 0;
    }
    return n_rest > 0 ? launch_pdl(attention_kernel<HD, 0>, dim3(n_rest), bd, AttnSmem<HD>::TOTAL, st, 1, pd)
                      : cudaSuccess;
}

}  // namespace

cudaError_t attention_launch(const AttnParams& p, cudaStream_t st) {
    static_assert(AttnSmem<128>::BAR_OFF - AttnSmem<128>::Q_BYTES >= kWarps * 16 * 128 * 4 + kWarps * 16 * 8,
                  "key-mode merge scratch must fit in the K/V stages");
    if (p.head_dim == 128) return launch_hd<128>(p, st);
    if (p.head_dim == 64) return launch_hd<64>(p, st);
    return cudaErrorInvalidValue;
}

cudaError_t attention_combine_launch(const AttnParams& p, cudaStream_t st) {
    if (p.n_combines == 0) return cudaSuccess;
    if (p.head_dim == 128) return launch_pdl(attention_combine_kernel<128>, dim3(p.n_combines), dim3(256), 0, st, 1, p);
    if (p.head_dim == 64) return launch_pdl(attention_combine_kernel<64>, dim3(p.n_combines), dim3(256), 0, st, 1, p);
    return cudaErrorInvalidValue;
}

}  // namespace ssk
