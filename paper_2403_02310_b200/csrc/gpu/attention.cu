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
//             walks the whole key range; classic flash-attention-2 loop.
//   key mode  (rows <= 16, decodes):      all warps share the rows; each warp
//             takes a 16-key slice of every 64-key tile, and the four partial
//             softmax states are merged in shared memory at the end.
// Long key ranges are split across CTAs (split-KV); partial (m, l, O) go to a
// workspace and attention_combine merges them in a fixed order (deterministic).
//
// K/V pages ([block][kv_head][16][hd], 4 KB contiguous per page at hd=128) are
// streamed with cp.async into an XOR-swizzled double buffer; S = QK^T and
// O += PV use mma.sync m16n8k16 (bf16 in, fp32 accumulate).
#include <cfloat>

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
    static constexpr int ROW_BYTES = HD * 2;
    static constexpr int CHUNKS = HD / 8;  // 16 B chunks per row
    static constexpr int Q_BYTES = kRowsPerTile * ROW_BYTES;
    static constexpr int KV_TILE = kKeysPerTile * ROW_BYTES;
    static constexpr int STAGE = 2 * KV_TILE;  // K + V
    static constexpr int TOTAL = Q_BYTES + kStages * STAGE;
};

// byte offset of (row, 16B chunk c) in an XOR-swizzled tile
template <int HD>
__device__ __forceinline__ uint32_t swz(int row, int c) {
    return uint32_t(row * (HD * 2) + ((c ^ (row & 7)) << 4));
}

template <int HD>
__device__ __forceinline__ void load_kv_tile(const AttnParams& p, uint8_t* sK, uint8_t* sV, int e, int h, int kbase,
                                             int key1) {
    constexpr int CH = HD / 8;
    const int32_t* bt = p.block_table + size_t(e) * p.max_blocks;
    const size_t page = size_t(16) * HD;  // elements per (block, head) page
    for (int idx = threadIdx.x; idx < kKeysPerTile * CH; idx += kWarps * 32) {
        const int r = idx / CH, c = idx % CH;
        const int key = kbase + r;
        const uint32_t so = swz<HD>(r, c);
        if (key < key1) {
            const int32_t blk = bt[key >> 4];
            const size_t off = (size_t(blk) * p.nkv_l + h) * page + size_t(key & 15) * HD + c * 8;
            cp_async16(smem_u32(sK) + so, p.kc + off);
            cp_async16(smem_u32(sV) + so, p.vc + off);
        } else {
            cp_async_zero16(smem_u32(sK) + so, p.kc);
            cp_async_zero16(smem_u32(sV) + so, p.vc);
        }
    }
}

// KPW = keys handled per warp per 64-key tile (64: row mode, 16: key mode).
template <int HD, int KPW>
__device__ __forceinline__ void attend(const AttnParams& p, const AttnItem& it, uint8_t* smem, int qrow_base,
                                       int kofs, float (&O)[HD / 8][4], float (&m)[2], float (&l)[2]) {
    using S = AttnSmem<HD>;
    constexpr int NT = KPW / 8;  // n8 tiles of S per warp
    const int lane = threadIdx.x & 31;
    uint8_t* sQ = smem;
    const int e = it.entry;
    const int tok0 = p.cu_q[e];
    const int ntok = p.cu_q[e + 1] - tok0;
    const int prefix = p.ctx_len[e] - ntok;

    // Q fragments for this warp's 16 rows, all HD/16 k-steps.
    uint32_t qa[HD / 16][4];
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
        const int r = qrow_base + (lane & 15);
        ldsm_x4(smem_u32(sQ) + swz<HD>(r, ks * 2 + (lane >> 4)), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    }
    // causal limits of the two rows this thread holds
    int lim[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int r = qrow_base + (lane >> 2) + hr * 8;
        lim[hr] = r < it.nrows ? prefix + (it.row0 + r) / p.group : -1;
    }
    m[0] = m[1] = -INFINITY;
    l[0] = l[1] = 0.f;
#pragma unroll
    for (int dt = 0; dt < HD / 8; ++dt) O[dt][0] = O[dt][1] = O[dt][2] = O[dt][3] = 0.f;

    const int ntiles = (it.key1 - it.key0 + kKeysPerTile - 1) / kKeysPerTile;
    // kStages-deep cp.async ring: kStages-1 tiles stay in flight while one is consumed
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < ntiles) {
            uint8_t* nK = smem + S::Q_BYTES + s * S::STAGE;
            load_kv_tile<HD>(p, nK, nK + S::KV_TILE, e, it.kv_head, it.key0 + s * kKeysPerTile, it.key1);
        }
        cp_async_commit();
    }
    for (int t = 0; t < ntiles; ++t) {
        const int kbase = it.key0 + t * kKeysPerTile;
        uint8_t* sK = smem + S::Q_BYTES + (t % kStages) * S::STAGE;
        uint8_t* sV = sK + S::KV_TILE;
        if (t + kStages - 1 < ntiles) {
            uint8_t* nK = smem + S::Q_BYTES + ((t + kStages - 1) % kStages) * S::STAGE;
            load_kv_tile<HD>(p, nK, nK + S::KV_TILE, e, it.kv_head, kbase + (kStages - 1) * kKeysPerTile, it.key1);
        }
        cp_async_commit();
        cp_async_wait<kStages - 1>();
        __syncthreads();

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
                ldsm_x4(smem_u32(sK) + swz<HD>(key, ks * 2 + ((lane >> 3) & 1)), b0, b1, b2, b3);
                mma_bf16_16816(s[nt], qa[ks], b0, b1);
                mma_bf16_16816(s[nt + 1], qa[ks], b2, b3);
            }
        }
        // mask, online softmax (log2 domain)
        float mt[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int key = kbase + kofs + nt * 8 + 2 * (lane & 3) + (c & 1);
                const int hr = c >> 1;
                const bool vis = key <= lim[hr] && key < it.key1;
                s[nt][c] = vis ? s[nt][c] * p.scale_log2 : -INFINITY;
                mt[hr] = fmaxf(mt[hr], s[nt][c]);
            }
        }
        float alpha[2], msub[2];
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            mt[hr] = fmaxf(mt[hr], __shfl_xor_sync(0xffffffffu, mt[hr], 1));
            mt[hr] = fmaxf(mt[hr], __shfl_xor_sync(0xffffffffu, mt[hr], 2));
            const float mn = fmaxf(m[hr], mt[hr]);
            msub[hr] = mn == -INFINITY ? 0.f : mn;
            alpha[hr] = exp2f(m[hr] - msub[hr]);
            m[hr] = mn;
            l[hr] *= alpha[hr];
        }
#pragma unroll
        for (int dt = 0; dt < HD / 8; ++dt) {
            O[dt][0] *= alpha[0];
            O[dt][1] *= alpha[0];
            O[dt][2] *= alpha[1];
            O[dt][3] *= alpha[1];
        }
        uint32_t pa[NT / 2][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const float p0 = exp2f(s[nt][0] - msub[0]), p1 = exp2f(s[nt][1] - msub[0]);
            const float p2 = exp2f(s[nt][2] - msub[1]), p3 = exp2f(s[nt][3] - msub[1]);
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
                ldsm_x4_t(smem_u32(sV) + swz<HD>(key, dt + (lane >> 4)), b0, b1, b2, b3);
                mma_bf16_16816(O[dt], a, b0, b1);
                mma_bf16_16816(O[dt + 1], a, b2, b3);
            }
        }
        __syncthreads();  // this stage is refilled by a later iteration's prefetch
    }
    cp_async_wait<0>();
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        l[hr] += __shfl_xor_sync(0xffffffffu, l[hr], 1);
        l[hr] += __shfl_xor_sync(0xffffffffu, l[hr], 2);
    }
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
        float* po = p.part_o + size_t(it.part + r) * HD + d;
        po[0] = o0;
        po[1] = o1;
        if (d == 0) {
            p.part_ml[size_t(it.part + r) * 2 + 0] = mm;
            p.part_ml[size_t(it.part + r) * 2 + 1] = ll;
        }
    }
}

template <int HD>
__global__ void __launch_bounds__(kWarps * 32) attention_kernel(const AttnParams p) {
    using S = AttnSmem<HD>;
    extern __shared__ __align__(128) uint8_t smem[];
    const AttnItem it = p.items[blockIdx.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool key_mode = it.nrows <= 16;

    // stage the Q tile (rows beyond nrows are zero)
    {
        constexpr int CH = HD / 8;
        const int e = it.entry, tok0 = p.cu_q[e];
        const int nr = key_mode ? 16 : kRowsPerTile;
        for (int idx = threadIdx.x; idx < nr * CH; idx += kWarps * 32) {
            const int r = idx / CH, c = idx % CH;
            const uint32_t so = smem_u32(smem) + swz<HD>(r, c);
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
        return;
    }

    attend<HD, 16>(p, it, smem, 0, warp * 16, O, m, l);
    // merge the four warps' partial softmax states (smem reused after the loop)
    __syncthreads();
    float* sO = reinterpret_cast<float*>(smem + S::Q_BYTES);  // [4][16][HD]
    float* sML = sO + kWarps * 16 * HD;                        // [4][16][2]
    {
        const int r0 = lane >> 2;
#pragma unroll
        for (int dt = 0; dt < HD / 8; ++dt) {
            const int d = dt * 8 + 2 * (lane & 3);
            sO[(warp * 16 + r0) * HD + d] = O[dt][0];
            sO[(warp * 16 + r0) * HD + d + 1] = O[dt][1];
            sO[(warp * 16 + r0 + 8) * HD + d] = O[dt][2];
            sO[(warp * 16 + r0 + 8) * HD + d + 1] = O[dt][3];
        }
        if ((lane & 3) == 0) {
            sML[(warp * 16 + r0) * 2] = m[0];
            sML[(warp * 16 + r0) * 2 + 1] = l[0];
            sML[(warp * 16 + r0 + 8) * 2] = m[1];
            sML[(warp * 16 + r0 + 8) * 2 + 1] = l[1];
        }
    }
    __syncthreads();
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
            o0 += sO[(w * 16 + r) * HD + d] * f;
            o1 += sO[(w * 16 + r) * HD + d + 1] * f;
        }
        emit_pair<HD>(p, it, r, d, o0, o1, M, L);
    }
}

template <int HD>
__global__ void attention_combine_kernel(const AttnParams p) {
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
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(attention_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             AttnSmem<HD>::TOTAL);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (p.n_items > 0) attention_kernel<HD><<<p.n_items, kWarps * 32, AttnSmem<HD>::TOTAL, st>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t attention_launch(const AttnParams& p, cudaStream_t st) {
    static_assert(AttnSmem<128>::TOTAL >= AttnSmem<128>::Q_BYTES + kWarps * 16 * 128 * 4 + kWarps * 16 * 8,
                  "key-mode merge scratch must fit in the KV stages");
    if (p.head_dim == 128) return launch_hd<128>(p, st);
    if (p.head_dim == 64) return launch_hd<64>(p, st);
    return cudaErrorInvalidValue;
}

cudaError_t attention_combine_launch(const AttnParams& p, cudaStream_t st) {
    if (p.n_combines == 0) return cudaSuccess;
    if (p.head_dim == 128) attention_combine_kernel<128><<<p.n_combines, 256, 0, st>>>(p);
    else if (p.head_dim == 64) attention_combine_kernel<64><<<p.n_combines, 256, 0, st>>>(p);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace ssk
