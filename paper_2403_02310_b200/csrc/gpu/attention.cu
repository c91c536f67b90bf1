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
// K/V pages ([block][kv_head][16][hd], 4 KB contiguous at hd=128) are moved by
// TMA (cp.async.bulk.tensor, SWIZZLE_128B) into a kStages-deep full/empty
// mbarrier ring by a dedicated producer warp: no per-thread address math or
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

template <int HD>
struct AttnSmem {
    static constexpr int Q_BYTES = kRowsPerTile * HD * 2;
    static constexpr int KV_TILE = kKeysPerTile * HD * 2;  // [HD/64 halves][64 keys][128 B]
    static constexpr int STAGE = 2 * KV_TILE;              // K + V
    static constexpr int BAR_OFF = Q_BYTES + kStages * STAGE;
    // 896 B of alignment slack (the dynamic window starts 1 KB-aligned in practice;
    // checked at run time) keeps two CTAs per SM within 228 KB at hd = 128
    static constexpr int TOTAL = BAR_OFF + 64 + 896;
};

// Q tile: rows of HD*2 bytes, 16-byte chunks XOR-swizzled by row.
template <int HD>
__device__ __forceinline__ uint32_t swz_q(int row, int c) {
    return uint32_t(row * (HD * 2) + ((c ^ (row & 7)) << 4));
}
// K/V tile as written by TMA with SWIZZLE_128B: [c / 8 half][key][128 B].
__device__ __forceinline__ uint32_t swz_kv(int key, int c) {
    return uint32_t((c >> 3) * (kKeysPerTile * 128) + key * 128 + (((c & 7) ^ (key & 7)) << 4));
}

template <int HD>
__device__ __forceinline__ void issue_kv_tile(const AttnParams& p, const CUtensorMap* tmK, const CUtensorMap* tmV,
                                              uint8_t* sK, uint8_t* sV, uint64_t* bar, int e, int h, int kbase) {
    const int32_t* bt = p.block_table + size_t(e) * p.max_blocks;
    const int nvalid = (p.ctx_len[e] + 15) >> 4;
    mbar_arrive_expect_tx(bar, 2 * AttnSmem<HD>::KV_TILE);
#pragma unroll
    for (int pg = 0; pg < kKeysPerTile / 16; ++pg) {
        const int lb = (kbase >> 4) + pg;
        // pages past the context are masked; point them at a valid (finite) page
        const int32_t blk = bt[lb < nvalid ? lb : 0];
        const int32_t row = int32_t(p.layer_row0 + (int64_t(blk) * p.nkv_l + h) * 16);
#pragma unroll
        for (int hh = 0; hh < HD / 64; ++hh) {
            const uint32_t off = uint32_t(hh * (kKeysPerTile * 128) + pg * 16 * 128);
            tma_load_2d(sK + off, tmK, hh * 64, row, bar);
            tma_load_2d(sV + off, tmV, hh * 64, row, bar);
        }
    }
}

// KPW = keys handled per warp per 64-key tile (64: row mode, 16: key mode).
template <int HD, int KPW>
__device__ __forceinline__ void attend(const AttnParams& p, const CUtensorMap* tmK, const CUtensorMap* tmV,
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

    uint64_t* empty = full + kStages;
    const int ntiles = (it.key1 - it.key0 + kKeysPerTile - 1) / kKeysPerTile;
    for (int t = 0; t < ntiles; ++t) {
        const int kbase = it.key0 + t * kKeysPerTile;
        const int st = t % kStages;
        uint8_t* sK = smem + S::Q_BYTES + st * S::STAGE;
        uint8_t* sV = sK + S::KV_TILE;
        mbar_wait(&full[st], uint32_t((t / kStages) & 1));

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

template <int HD>
__global__ void __launch_bounds__((kWarps + 1) * 32) attention_kernel(const AttnParams p,
                                                                      const __grid_constant__ CUtensorMap tmK,
                                                                      const __grid_constant__ CUtensorMap tmV) {
    using S = AttnSmem<HD>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t pad = ((raw + 1023u) & ~1023u) - raw;
    if (pad > 896u) __trap();  // SWIZZLE_128B tiles need 1 KB alignment
    uint8_t* smem = smem_raw + pad;
    const AttnItem it = p.items[blockIdx.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool key_mode = it.nrows <= 16;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
    uint64_t* empty = full + kStages;

    if (threadIdx.x == 0) {
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        mbar_fence_init();
    }
    pdl_launch_dependents();
    pdl_wait();  // q / KV of this layer come from the preceding kernels
    // stage the Q tile (rows beyond nrows are zero)
    {
        constexpr int CH = HD / 8;
        const int e = it.entry, tok0 = p.cu_q[e];
        const int nr = key_mode ? 16 : kRowsPerTile;
        for (int idx = threadIdx.x; idx < nr * CH; idx += (kWarps + 1) * 32) {
            const int r = idx / CH, c = idx % CH;
            const uint32_t so = smem_u32(smem) + swz_q<HD>(r, c);
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
        __syncthreads();
    }

    if (warp == kWarps) {  // ---- producer warp: K/V pages by TMA into the ring
        if (lane == 0) {
            const int ntiles = (it.key1 - it.key0 + kKeysPerTile - 1) / kKeysPerTile;
            for (int t = 0; t < ntiles; ++t) {
                const int st = t % kStages;
                if (t >= kStages) mbar_wait(&empty[st], uint32_t(((t / kStages) - 1) & 1));
                uint8_t* sk = smem + S::Q_BYTES + st * S::STAGE;
                issue_kv_tile<HD>(p, &tmK, &tmV, sk, sk + S::KV_TILE, &full[st], it.entry, it.kv_head,
                                  it.key0 + t * kKeysPerTile);
            }
        }
        return;
    }

    float O[HD / 8][4], m[2], l[2];
    if (!key_mode) {
        attend<HD, 64>(p, &tmK, &tmV, it, smem, warp * 16, 0, O, m, l);
        const int r0 = warp * 16 + (lane >> 2);
#pragma unroll
        for (int dt = 0; dt < HD / 8; ++dt) {
            const int d = dt * 8 + 2 * (lane & 3);
            emit_pair<HD>(p, it, r0, d, O[dt][0], O[dt][1], m[0], l[0]);
            emit_pair<HD>(p, it, r0 + 8, d, O[dt][2], O[dt][3], m[1], l[1]);
        }
        if (p.fused_combine) finish_split<HD>(p, it, reinterpret_cast<int*>(smem + S::BAR_OFF + 2 * kStages * 8));
        return;
    }

    attend<HD, 16>(p, &tmK, &tmV, it, smem, 0, warp * 16, O, m, l);
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
    if (p.fused_combine) finish_split<HD>(p, it, reinterpret_cast<int*>(smem + S::BAR_OFF + 2 * kStages * 8));
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
cudaError_t launch_hd(const AttnParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(attention_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             AttnSmem<HD>::TOTAL);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    return p.n_items > 0 ? launch_pdl(attention_kernel<HD>, dim3(p.n_items), dim3((kWarps + 1) * 32), AttnSmem<HD>::TOTAL,
                                      st, 1, p, tk, tv)
                         : cudaSuccess;
}

}  // namespace

bool attention_tmaps(CUtensorMap* tk, CUtensorMap* tv, const void* kc, const void* vc, int64_t total_rows, int hd) {
    return make_tmap_2d(tk, kc, uint64_t(total_rows), uint64_t(hd), 16, 64) &&
           make_tmap_2d(tv, vc, uint64_t(total_rows), uint64_t(hd), 16, 64);
}

cudaError_t attention_launch(const AttnParams& p, const CUtensorMap& tk, const CUtensorMap& tv, cudaStream_t st) {
    static_assert(AttnSmem<128>::BAR_OFF - AttnSmem<128>::Q_BYTES >= kWarps * 16 * 128 * 4 + kWarps * 16 * 8,
                  "key-mode merge scratch must fit in the K/V stages");
    if (p.head_dim == 128) return launch_hd<128>(p, tk, tv, st);
    if (p.head_dim == 64) return launch_hd<64>(p, tk, tv, st);
    return cudaErrorInvalidValue;
}

cudaError_t attention_combine_launch(const AttnParams& p, cudaStream_t st) {
    if (p.n_combines == 0) return cudaSuccess;
    if (p.head_dim == 128) return launch_pdl(attention_combine_kernel<128>, dim3(p.n_combines), dim3(256), 0, st, 1, p);
    if (p.head_dim == 64) return launch_pdl(attention_combine_kernel<64>, dim3(p.n_combines), dim3(256), 0, st, 1, p);
    return cudaErrorInvalidValue;
}

}  // namespace ssk
