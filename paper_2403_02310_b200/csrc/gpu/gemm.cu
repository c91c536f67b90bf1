// K3: projection GEMMs over the packed token dimension on 5th-gen tensor cores.
//
//   D[M, N] = A[M, K] . B[N, K]^T      A = activations (bf16, K-major)
//                                      B = weight shard (bf16, K-major)
//
// Persistent, warp-specialised tcgen05 kernel, one CTA per SM:
//   warp 0       TMA producer: A/B tiles (SWIZZLE_128B) into a STAGES-deep ring
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer (fp32
//                accumulators in TMEM, K = 16 per instruction)
//   warps 2..9   epilogue: tcgen05.ld -> registers -> fused epilogue -> HBM
//                (two warps per TMEM lane quarter, alternating 32-column chunks)
// CG = 2 runs CTA pairs (cluster of 2, tcgen05 cta_group::2): a 256 x BN tile
// per pair, each CTA staging its own 128 rows of A and BN/2 rows of B, so the
// per-SM shared-memory traffic per MMA is half that of a 1-CTA 128 x BN tile.
// The leader CTA issues the MMAs; smem-slot and accumulator barriers are
// multicast-committed to both CTAs. CG = 1 (128 x BN) serves small M (LM head,
// decode-only batches). Accumulators are double-buffered in TMEM so a tile's
// epilogue overlaps the next tile's MMAs. The M tail (T = 481, 2017, ...) is
// handled by TMA zero fill on load and row masking on store.
//
// Fused epilogues (K4 work folded into K3):
//   EPI_BF16    store bf16 D (QKV projection, TP partials)
//   EPI_RESADD  x_f32 += D   (O / down projections: residual add, TP = 1)
//   EPI_SWIGLU  gate/up rows interleaved in 32-row groups: out = silu(g) * u
//   EPI_F32     store fp32 D (LM head logits)
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace ssk {

namespace {

constexpr int BK = 64;  // 128 B of bf16: one SWIZZLE_128B row
constexpr int kThreads = 320;  // chain kernel: warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
// gemm_tcgen05_kernel: warp 0 TMA, warp 1 MMA, warps 2..3 register donors, warps 4..11 epilogue.
// Three warpgroups so the registers can be rebalanced with setmaxnreg (warpgroup-wide): the
// control warpgroup drops to kRegsCtl, the two epilogue warpgroups grow to kRegsEpi
// (per scheduler: one warp of each warpgroup; kRegsCtl + 2 kRegsEpi must fit the 3 x 168
// allocated at launch, or the increase never completes), instead of every
// warp being capped at 168 and the epilogue's residual / RoPE operands spilling to memory.
constexpr int kGemmThreads = 384;
constexpr int kRegsCtl = 88, kRegsEpi = 208;
static_assert(kRegsCtl + 2 * kRegsEpi <= 3 * 168, "setmaxnreg budget exceeds the launch allocation");
constexpr int kSmemMax = 232448;                         // 227 KB opt-in per CTA
constexpr int kSmemBudget = kSmemMax - 1024 - 1024 - 8 * 4096;  // operand ring

// AR < 128 (single-CTA tiles, M <= AR): only AR rows of A are loaded per stage; the MMA
// still reads 128 rows from the stage, the rest being whatever follows in smem, which only
// lands in accumulator rows >= M that are never stored. The freed smem buys more stages
// of weight tiles in flight (decode-only batches are weight-streaming bound per SM).
template <int CG, int BN, int AR = 128>
struct GemmCfg {
    static constexpr int A_BYTES = AR * BK * 2;        // this CTA's rows of A
    static constexpr int B_ROWS = BN / CG;             // this CTA's rows of B
    static constexpr int B_BYTES = B_ROWS * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES_FIT = kSmemBudget / STAGE_BYTES;
    // narrow weight-streaming tiles (decode-sized M) keep more, smaller stages in flight
#ifndef SS_GEMM_STAGES_CAP  // dev: cap the operand ring depth (latency-sensitivity probes)
#define SS_GEMM_STAGES_CAP 16
#endif
    static constexpr int STAGES_MAX = (STAGE_BYTES <= 16384 ? 16 : 8) < SS_GEMM_STAGES_CAP
                                          ? (STAGE_BYTES <= 16384 ? 16 : 8)
                                          : SS_GEMM_STAGES_CAP;
    static constexpr int STAGES = STAGES_FIT > STAGES_MAX ? STAGES_MAX : STAGES_FIT;
    static constexpr int TMEM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
    // + barriers (1 KB slot) + the epilogue warps' 4 KB staging buffers
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 1024 + 8 * 4096;
    static_assert(SMEM <= kSmemMax, "shared memory over the per-CTA limit");
    static constexpr int TILE_M = 128 * CG;
};

// fast reciprocal division: the product is rounded to bf16 anyway
__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
// Wait that acquires at cluster scope: the phase was completed by another CTA's arrive.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0, spins = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (++spins == (1u << 28)) __trap();
    }
}
// Bulk copy from this CTA's shared memory into another cluster CTA's, completing on that
// CTA's mbarrier (both cluster addresses from peer_addr).
__device__ __forceinline__ void bulk_s2cluster(uint32_t dst_cluster, const void* src, uint32_t bytes,
                                               uint32_t bar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst_cluster), "r"(smem_u32(src)), "r"(bytes), "r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Relaxed arrive: orders nothing but the (tcgen05-fenced) TMEM reads, so the
// epilogue's global stores need not drain before the accumulator is handed back.
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-SM TMA: data lands in this CTA, completion is signalled on the leader's mbarrier.
__device__ __forceinline__ void tma_load_2d_cg2(void* smem_dst, const CUtensorMap* m, int32_t c0, int32_t c1,
                                                uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar_cluster)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d_cg2_hint(void* smem_dst, const CUtensorMap* m, int32_t c0, int32_t c1,
                                                     uint32_t bar_cluster, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(policy)
        : "memory");
}

template <int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t* slot, uint32_t cols_pow2);
template <>
__device__ __forceinline__ void tmem_alloc_cg<1>(uint32_t* slot, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <>
__device__ __forceinline__ void tmem_alloc_cg<2>(uint32_t* slot, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t taddr, uint32_t cols) {
    if constexpr (CG == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
    else
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}
template <int CG>
__device__ __forceinline__ void mma_cg(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (CG == 1) {
        umma_bf16(d, a, b, idesc, acc);
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    }
}
// Commit: arrive on `bar` (same smem offset) in every CTA of the group once the
// issued MMAs retire.
template <int CG>
__device__ __forceinline__ void commit_cg(uint64_t* bar, uint16_t mask = 3) {
    if constexpr (CG == 1) {
        umma_commit(bar);
    } else {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(bar)),
            "h"(mask)
            : "memory");
    }
}
// 2-SM TMA multicast: this CTA's slice lands at the same smem offset in every CTA of `mask`;
// each destination's bytes complete on the barrier at this offset in its own pair leader.
__device__ __forceinline__ void tma_load_2d_cg2_mc_hint(void* smem_dst, const CUtensorMap* m, int32_t c0, int32_t c1,
                                                        uint32_t bar_cluster, uint16_t mask, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5, %6;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar_cluster), "h"(mask), "l"(policy)
        : "memory");
}

// One lane of the (fully active) warp: the issuer of single-thread tcgen05 ops.
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Stream-K split of the (tile, k-block) iteration space: group g of G owns the
// contiguous range [g*I/G, (g+1)*I/G). A range is walked as segments; a segment
// that starts a tile at k-block 0 but does not finish it is the tile's "head"
// and reduces the partial accumulators of the groups that hold the rest of the
// tile (each of them starts its range inside that tile and processes that piece
// first, so the head — processed last by its owner — never waits long).
struct SkRange {
    long i0, i1;
};
__device__ __forceinline__ SkRange sk_range(int gid, int G, long total) {
    return SkRange{long(gid) * total / G, long(gid + 1) * total / G};
}
__device__ __forceinline__ long sk_start(int g, int G, long total) { return long(g) * total / G; }

// Work segments of one group. mode 0: whole tiles round-robin (tile g, g+G, ...:
// concurrently active tiles are neighbours, so B/A tiles are shared in L2);
// mode 1: the group's stream-K range cut at tile boundaries.
// mode 3: M-lockstep stream-K. The groups form super-groups of P = num_mt
// consecutive groups, member m owning M-tile m; stream-K runs over the
// (N-tile, k-block) space of the super-groups, so the P members walk identical
// B k-blocks at the same time (each weight byte leaves HBM once, the P reads
// meet in L2) and every group gets the same number of k-blocks whatever the
// tile count — no wave quantisation for the under-filled M = 256..2048 shapes.
struct Seg {
    int t, kb0, kb1;
};
// mode 2: split-K in lockstep — S aligned K slices per tile, one (tile, slice)
// unit per group (units <= groups): group g runs slice g % S of tile g / S, so
// every group walks the same K offsets at the same time (A k-blocks shared in
// L2) and a tile's pieces sit on consecutive groups.
struct SegIter {
    int mode, G, num_kb, num_tiles, t_rr, S, P, mem;
    long i, i1;
    __device__ SegIter(int m, int gid, int G_, int nkb, int nt, SkRange r, int S_, int P_)
        : mode(m), G(G_), num_kb(nkb), num_tiles(nt), t_rr(gid), S(S_), P(P_), mem(gid % P_), i(r.i0), i1(r.i1) {}
    __device__ __forceinline__ bool next(Seg& s) {
        if (mode == 0) {
            if (t_rr >= num_tiles) return false;
            s = Seg{t_rr, 0, num_kb};
            t_rr += G;
            return true;
        }
        if (mode == 2) {
            // whole tiles for the full waves, then the ragged last wave split in
            // S aligned K slices (one unit per group, consecutive groups per tile)
            const int full = (num_tiles / G) * G;
            if (t_rr < full) {
                s = Seg{t_rr, 0, num_kb};
                t_rr += G;
                return true;
            }
            if (t_rr >= (1 << 29)) return false;
            const int u = t_rr - full - (t_rr - full) / G * G;  // == gid
            t_rr = 1 << 29;
            if (u >= (num_tiles - full) * S) return false;
            const int sl = u % S;
            s = Seg{full + u / S, sl * num_kb / S, (sl + 1) * num_kb / S};
            return true;
        }
        if (i >= i1) return false;
        s.t = int(i / num_kb) * P + mem;  // mode 3: N-tile i / num_kb, this member's M-tile
        s.kb0 = int(i % num_kb);
        s.kb1 = int(s.kb0 + (i1 - i) < num_kb ? s.kb0 + (i1 - i) : num_kb);
        i += s.kb1 - s.kb0;
        return true;
    }
};

#ifdef SS_GEMM_TRACE
// Dev-only timeline (build with -DSS_GEMM_TRACE): per CTA, globaltimer ns at
// entry, after pdl_wait, first full stage, last MMA of the first segment,
// accumulator seen by the epilogue, first segment stored, exit.
__device__ unsigned long long g_gemm_trace[1024][8];
__device__ int g_trace_epi = -1;  // >= 0: record only launches with this epilogue
__device__ __forceinline__ void trace(int i) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_gemm_trace[blockIdx.x][i] = t;
}
__device__ unsigned long long g_gemm_trace2[1024][16];
__device__ __forceinline__ void trace2(int i) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_gemm_trace2[blockIdx.x][i] = t;
}
#define TRACE(i) \
    if (g_trace_epi < 0 || g_trace_epi == EPI) trace(i)
#define TRACE2(i) \
    if (warp == (blockDim.x == kGemmThreads ? 4 : 2) && lane == 0 && (g_trace_epi < 0 || g_trace_epi == EPI)) trace2(i)
#else
#define TRACE(i)
#define TRACE2(i)
#endif

// ---- staged split-K fixup (last segment of a group: the smem ring is idle)
// Partial layout per (group, CTA rank): [chunk c][row 0..127][32 fp32], a warp's
// 32 rows of one chunk = 4 KB contiguous, float4 j of row r at slot j ^ (r & 7)
// (conflict-free smem reads for the 8 lanes of a quarter-warp).
__device__ __forceinline__ void bulk_store_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_all() {
    asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
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
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Per-warp epilogue staging buffer: 32 rows x 128 B, 16-byte chunk j of row r at
// slot r * 8 + (j ^ (r & 7)). stage_rows writes this thread's row (thread = row);
// add_rows adds the staged fp32 row to v.
__device__ __forceinline__ void stage_rows(uint4* ep, const uint32_t (&v)[32], int lane) {
#pragma unroll
    for (int j = 0; j < 8; ++j) ep[lane * 8 + (j ^ (lane & 7))] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}
__device__ __forceinline__ void add_rows(uint32_t (&v)[32], const uint4* ep, int lane) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint4 a = ep[lane * 8 + (j ^ (lane & 7))];
        v[4 * j + 0] = __float_as_uint(__uint_as_float(v[4 * j + 0]) + __uint_as_float(a.x));
        v[4 * j + 1] = __float_as_uint(__uint_as_float(v[4 * j + 1]) + __uint_as_float(a.y));
        v[4 * j + 2] = __float_as_uint(__uint_as_float(v[4 * j + 2]) + __uint_as_float(a.z));
        v[4 * j + 3] = __float_as_uint(__uint_as_float(v[4 * j + 3]) + __uint_as_float(a.w));
    }
}

// MC = 2 (CG = 2 only): clusters of two CTA pairs that walk identical weight (B) k-blocks
// (the two M-tile members of an M-lockstep stream-K super-group, or the two M-tiles of one
// column in the whole-tile schedule with an even M-tile count). Each CTA loads half of its
// B rows and multicasts them to its counterpart in the other pair, so every weight byte
// crosses the L2 -> SM fabric once per cluster instead of once per pair (the main loop is
// bound by that fabric when all pairs run, scripts/gemm_scaling.py). Both pairs' MMA
// commits release a stage in all four CTAs (empty barriers count two arrivals).
template <int CG, int BN, int EPI, int AR, int MC = 1>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M_rows,
                        int row0, int N, int K, void* __restrict__ out, int ldo, int num_mt, int num_tiles,
                        float* __restrict__ part, uint32_t* __restrict__ flags, uint32_t epoch, int sk_mode,
                        int sk_slices, int dsm, const EpiArgs ea) {
    using Cfg = GemmCfg<CG, BN, AR>;
    constexpr int STAGES = Cfg::STAGES;
    // rows [row0, row0 + M_rows) of A / the output / every row-indexed epilogue operand
    const int M = row0 + M_rows;  // exclusive row end
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* ebar = tempty + 2;  // one per epilogue warp (staged fixup loads)
    if constexpr (CG == 2) dsm = 0;  // cluster split-K is single-CTA only: fold its paths away
    uint64_t* gobar = ebar + 8;   // dsm: per epilogue warp, slice 0 opened its receive buffers
    uint64_t* donebar = gobar + 8;  // dsm: per epilogue warp, slice 0 holds this slice's partial
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(donebar + 8);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int num_kb = (K + BK - 1) / BK;
    const uint32_t crank = CG == 2 ? cluster_rank() : 0;  // rank in the cluster (MC pairs)
    const uint32_t rank = crank & 1u;                    // rank in the CTA pair
    const uint32_t pidx = crank >> 1;                    // pair in the cluster (MC = 2)
    const uint32_t lead_rank = crank & ~1u;
    const uint16_t pair_mask = uint16_t(3u << (2 * pidx));
    const uint16_t empty_mask = MC == 2 ? uint16_t(0xF) : pair_mask;
    const uint16_t b_mask = uint16_t((1u << rank) | (1u << (2 + rank)));  // MC = 2: this rank in both pairs
    const bool leader = rank == 0;
    const int gid = blockIdx.x / CG, G = gridDim.x / CG;
    // stream-K super-group size (mode 3: one member per M-tile; else 1)
    const int P = sk_mode == 3 ? num_mt : 1;
    const long total = long(num_tiles / P) * num_kb;
    const SkRange rg = sk_range(gid / P, G / P, total);
    if (threadIdx.x == 0) TRACE(0);

    if (threadIdx.x == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], MC);  // MC = 2: both pairs' MMAs released the stage
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8 * CG);  // every epilogue warp of the group
        }
        for (int a = 0; a < 8; ++a) {
            mbar_init(&ebar[a], 1);
            mbar_init(&gobar[a], 1);
            mbar_init(&donebar[a], 1);
        }
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc_cg<CG>(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    if (CG == 2 || dsm > 1) cluster_sync();  // dsm: barriers initialised before any remote arrive
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_launch_dependents();
    if constexpr (EPI == EPI_QKV) {
        if (sk_mode == 0 && gid >= num_tiles) {  // no tile for this pair: warm L2 for attention
            // (the cached pages are final: no kernel of this step writes them before attention)
            const int nthreads = (G - num_tiles) * CG * kGemmThreads;
            const int tid = ((gid - num_tiles) * CG + int(rank)) * kGemmThreads + int(threadIdx.x);
            const size_t page = size_t(ea.bs) * ea.hd;  // elements of one (block, head) page
            for (int w = tid; w < ea.pf_n * ea.pf_pages * 2; w += nthreads) {
                const int i = w / (ea.pf_pages * 2), pg = (w >> 1) % ea.pf_pages, kv = w & 1;
                const AttnItem itm = ea.pf_items[i];
                const int lb = (itm.key0 >> 4) + pg;
                if (lb * ea.bs >= itm.key1 || lb * ea.bs >= ea.pf_ctx_len[itm.entry]) continue;
                const int32_t blk = ea.pf_bt[size_t(itm.entry) * ea.pf_max_blocks + lb];
                const __nv_bfloat16* src = (kv ? ea.vc : ea.kc) + (size_t(blk) * ea.nkv + itm.kv_head) * page;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(uint32_t(page * 2))
                             : "memory");
            }
        }
    }
    // Programmatic dependent launch: A (activations) and the residual come from the
    // preceding kernels, so the producer and the epilogue warps wait for them; the
    // MMA warp only consumes shared memory and needs no wait.

    // the register file is rebalanced per role (setmaxnreg at the head of each branch):
    // control warpgroup (warps 0..3) down to kRegsCtl, epilogue warpgroups up to kRegsEpi
    if (warp == 0) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl));
        if (lane == 0) {  // ---------------- TMA producer (both CTAs)
            const uint32_t full_leader = CG == 2 ? peer_addr(full, lead_rank) : 0;
            // MC = 2: this CTA's half of its B rows, multicast to its counterpart
            constexpr int B_LOAD_ROWS = Cfg::B_ROWS / MC;
            const int b_half = MC == 2 ? int(pidx) * B_LOAD_ROWS : 0;
            const uint64_t polA = (ea.l2hint & 1) ? l2_policy_evict_last() : l2_policy_evict_normal();
            const uint64_t polB = (ea.l2hint & 2) ? l2_policy_evict_first() : l2_policy_evict_normal();
            // The weights (B) do not depend on the preceding kernels: the first
            // stages' B tiles are requested before the grid-dependency wait, so
            // their HBM latency overlaps the previous kernel's tail.
            int npre = 0;
            {
                SegIter pit(sk_mode, gid, G, num_kb, num_tiles, rg, sk_slices, P);
                Seg sg;
                if (pit.next(sg)) {
                    const int n0 = (sg.t / num_mt) * BN + Cfg::B_ROWS * int(rank);
                    npre = sg.kb1 - sg.kb0 < STAGES ? sg.kb1 - sg.kb0 : STAGES;
                    for (int j = 0; j < npre; ++j) {
                        const int kb = sg.kb0 + j;
                        if constexpr (CG == 1) {
                            mbar_arrive_expect_tx(&full[j], Cfg::STAGE_BYTES);
                            tma_load_2d_hint(sB + j * Cfg::B_BYTES, &tmB, kb * BK, n0, &full[j], polB);
                        } else {
                            if (leader) mbar_arrive_expect_tx(&full[j], 2 * Cfg::STAGE_BYTES);
                            if constexpr (MC == 2)
                                tma_load_2d_cg2_mc_hint(sB + j * Cfg::B_BYTES + b_half * 128, &tmB, kb * BK, n0 + b_half,
                                                        full_leader + uint32_t(j * 8), b_mask, polB);
                            else
                                tma_load_2d_cg2_hint(sB + j * Cfg::B_BYTES, &tmB, kb * BK, n0, full_leader + uint32_t(j * 8), polB);
                        }
                    }
                }
            }
            pdl_wait();
            TRACE(1);
            int s = 0, it = 0;
            uint32_t ph = 0;
            SegIter sit(sk_mode, gid, G, num_kb, num_tiles, rg, sk_slices, P);
            for (Seg sg; sit.next(sg);) {
                const int t = sg.t, kb0 = sg.kb0, kb1 = sg.kb1;
                const int m0 = row0 + (t % num_mt) * Cfg::TILE_M + 128 * int(rank);
                const int n0 = (t / num_mt) * BN + Cfg::B_ROWS * int(rank);
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const bool pre = it < npre;  // B already in flight, slot fresh
                    if (!pre) mbar_wait(&empty[s], ph ^ 1);
#if defined(SS_GEMM_EXP) && SS_GEMM_EXP == 1  // dev experiment: no loads (MMA on stale smem)
                    if (leader) mbar_arrive(&full[s]);
                    if (false)
#endif
                    if constexpr (CG == 1) {
                        if (!pre) {
                            mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
                            tma_load_2d_hint(sB + s * Cfg::B_BYTES, &tmB, kb * BK, n0, &full[s], polB);
                        }
                        tma_load_2d_hint(sA + s * Cfg::A_BYTES, &tmA, kb * BK, m0, &full[s], polA);
                    } else {
                        const uint32_t fb = full_leader + uint32_t(s * 8);
                        if (!pre) {
                            if (leader) mbar_arrive_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
                            if constexpr (MC == 2)
                                tma_load_2d_cg2_mc_hint(sB + s * Cfg::B_BYTES + b_half * 128, &tmB, kb * BK, n0 + b_half,
                                                        fb, b_mask, polB);
                            else
                                tma_load_2d_cg2_hint(sB + s * Cfg::B_BYTES, &tmB, kb * BK, n0, fb, polB);
                        }
                        tma_load_2d_cg2_hint(sA + s * Cfg::A_BYTES, &tmA, kb * BK, m0, fb, polA);
                    }
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl));
        // ---------------- MMA issuer (leader CTA only). The whole warp walks the
        // schedule converged, so descriptors and counters are warp-uniform and
        // live in uniform registers; one elected lane issues MMAs and commits
        // (a lone-lane issuer compiles to a per-MMA waterfall of R2UR moves that
        // starves the tensor core on narrow tiles).
        if (leader) {
            constexpr uint32_t idesc = umma_idesc_bf16(Cfg::TILE_M, BN);
            const uint64_t adesc0 = umma_desc_sw128(smem_u32(sA)), bdesc0 = umma_desc_sw128(smem_u32(sB));
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t acc_ph = 0;
            SegIter sit(sk_mode, gid, G, num_kb, num_tiles, rg, sk_slices, P);
#ifdef SS_GEMM_TRACE
            int seg_no = 0;
#endif
            for (Seg sg; sit.next(sg);) {
                const int kb0 = sg.kb0, kb1 = sg.kb1;
                mbar_wait(&tempty[acc], acc_ph ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
                const int nk = kb1 - kb0;
                for (int i = 0; i < nk; ++i) {
                    mbar_wait(&full[s], ph);  // TMA (async proxy) -> MMA (async proxy): no fence
#ifdef SS_GEMM_TRACE
                    if (i == 0 && seg_no == 0 && lane == 0) TRACE(2);
#endif
                    // descriptor start field is addr >> 4: stage / K-step offsets add directly
                    const uint64_t ad = adesc0 + uint64_t((s * Cfg::A_BYTES) >> 4);
                    const uint64_t bd = bdesc0 + uint64_t((s * Cfg::B_BYTES) >> 4);
                    if (elect_one()) {
#if !(defined(SS_GEMM_EXP) && SS_GEMM_EXP == 2)  // dev experiment 2: loads only
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            mma_cg<CG>(d_tmem, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc,
                                       (i > 0 || k > 0) ? 1u : 0u);
#endif
                        commit_cg<CG>(&empty[s], empty_mask);  // slot free (in both CTAs) once these MMAs retire
                    }
                    __syncwarp();
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (elect_one()) commit_cg<CG>(&tfull[acc], pair_mask);  // accumulator ready for both CTAs' epilogues
                __syncwarp();
#ifdef SS_GEMM_TRACE
                if (seg_no < 4 && lane == 0) TRACE(3 + seg_no);
                ++seg_no;
#endif
                if (++acc == 2) {
                    acc = 0;
                    acc_ph ^= 1;
                }
            }
        }
    } else if (warp < 4) {  // register donors
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl));
    } else {  // ---------------------------- epilogue warps 4..11
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsEpi));
        pdl_wait();
        // two warps per TMEM lane quarter (warp % 4 selects the quarter), splitting
        // the tile's 32-column chunks (pairs for SwiGLU) between them
        const int q = warp & 3;
        const int ew = warp - 4, half = ew >> 2;
        const uint32_t tempty_leader = CG == 2 ? peer_addr(tempty, lead_rank) : 0;
        const int rloc = 128 * int(rank) + q * 32 + lane;  // row within the group's tile
        // Stores leave through a per-warp 4 KB staging buffer: the accumulator arrives
        // one row per thread (tcgen05.ld 32x32b), is written to smem as 32 rows x 128 B
        // (16-byte chunks XOR-swizzled by row: conflict-free both ways) and read back
        // warp-coalesced (lane l of step j: row 4j + l/8, chunk l%8), so every global
        // access covers whole 32-byte sectors of few lines instead of one 16-byte
        // piece of 32 different lines.
        uint4* ep = reinterpret_cast<uint4*>(smem + STAGES * Cfg::STAGE_BYTES + 1024 + ew * 4096);
        const int crow = lane >> 3, cch = lane & 7;  // coalesced layout: row-in-step, chunk
        int acc = 0;
        uint32_t acc_ph = 0, eph = 0;
        SegIter sit(sk_mode, gid, G, num_kb, num_tiles, rg, sk_slices, P);
        // flag epoch of this launch (after pdl_wait: the forward's base is final)
        if (ea.epoch_base) epoch += *reinterpret_cast<const volatile uint32_t*>(ea.epoch_base);
        for (Seg sg; sit.next(sg);) {
            const int t = sg.t, kb0 = sg.kb0, kb1 = sg.kb1;
            const int m0 = row0 + (t % num_mt) * Cfg::TILE_M, n0 = (t / num_mt) * BN;
            const int row = m0 + rloc;
            const int rbase = row - lane;  // first row of this warp
            // RMSNorm of the A row, folded in: scale = rsqrt(mean(x^2) + eps). The
            // sums of squares come from the previous kernel, so this overlaps the
            // tile's main loop (computed before waiting for the accumulator). Loads are
            // coalesced (lane l takes float4 l, l + 32, ... of each of the warp's rows);
            // a 31-shuffle transpose-reduce leaves row `lane`'s total in lane `lane`.
            float rs = 1.f;
            if (ea.ssq_in && kb0 == 0) {
                const int n4 = ea.ssq_in_n >> 2;
                float a[32];
#pragma unroll
                for (int r = 0; r < 32; ++r) a[r] = 0.f;
                for (int i = lane; i - lane < n4; i += 32) {  // warp-uniform trip count
                    // 32 independent loads in flight per step (one per row)
#pragma unroll
                    for (int r = 0; r < 32; ++r) {
                        if (i < n4 && rbase + r < M) {
                            // volatile: issued here, before the accumulator wait, not sunk to the use
                            float4 w;
                            asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
                                         : "=f"(w.x), "=f"(w.y), "=f"(w.z), "=f"(w.w)
                                         : "l"(reinterpret_cast<const float4*>(ea.ssq_in + size_t(rbase + r) * ea.ssq_in_n) + i));
                            a[r] += (w.x + w.y) + (w.z + w.w);
                        }
                    }
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    const bool up = lane & off;
#pragma unroll
                    for (int i = 0; i < off; ++i) {
                        const float send = up ? a[i] : a[i + off];
                        const float keep = up ? a[i + off] : a[i];
                        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                    }
                }
                rs = rsqrtf(a[0] * ea.inv_dim + ea.eps);
            }
            // residual of this warp's first two chunks (coalesced layout), loaded
            // while the MMAs run
            float4 xin[2][8];
            if constexpr (EPI == EPI_RESADD) {
                if (kb0 == 0) {
                    // the later chunks' residual lines (this lane's row) go to L2 now
                    for (int c2 = half + 4; c2 < BN / 32; c2 += 2)
                        if (row < M && n0 + c2 * 32 < N)
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(static_cast<const float*>(out) +
                                                                         size_t(row) * ldo + n0 + c2 * 32));
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int col = n0 + (half + 2 * i) * 32 + cch * 4;
                        if (half + 2 * i < BN / 32 && col < N) {
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const int r = rbase + 4 * j + crow;
                                if (r < M)  // volatile: issued before the accumulator wait
                                    asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                                                 : "=f"(xin[i][j].x), "=f"(xin[i][j].y), "=f"(xin[i][j].z), "=f"(xin[i][j].w)
                                                 : "l"(static_cast<const float*>(out) + size_t(r) * ldo + col));
                            }
                        }
                    }
                }
            }
            // QKV: this row's position/slot and its RoPE factors, also fetched while the
            // MMAs run. Every chunk pair of a warp sits at the same offset i0 inside its
            // head (pairs step by whole heads), so one set of factors serves them all;
            // volatile loads keep the compiler from sinking them past the wait.
            int q_pos = 0;
            int64_t q_slot = 0;
            float4 rc[16];
            if constexpr (EPI == EPI_QKV) {
                if (kb0 == 0 && row < M) {
                    q_pos = ea.pos[row];
                    q_slot = ea.slot[row];
                    // this warp's chunk pairs (2 pi, 2 pi + 1), pi = half, half + 2: 128 columns
                    // apart, so the same offset i0 inside their heads (hd = 64 or 128)
                    if (half < BN / 64) {
                        const int col = n0 + 2 * half * 32;
                        if (col < N) {
                            const float4* cs = reinterpret_cast<const float4*>(ea.rope + size_t(q_pos) * (ea.hd / 2) +
                                                                               (col % ea.hd) / 2);
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
                                             : "=f"(rc[j].x), "=f"(rc[j].y), "=f"(rc[j].z), "=f"(rc[j].w)
                                             : "l"(cs + j));
                        }
                    }
                }
            }
            mbar_wait(&tfull[acc], acc_ph);
            tc_fence_after();
            TRACE2(0);
            const uint32_t t_row = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
            SegIter peek = sit;
            Seg nx;
            const bool last_seg = !peek.next(nx);
            constexpr int kStg = ((BN / 32 + 1) / 2) * 1024;  // staging floats per epilogue warp
            float* stg = reinterpret_cast<float*>(smem) + ew * kStg;
            // dsm > 1: this tile's dsm K slices are one thread-block cluster (slice = rank, one
            // segment per CTA, rows in TMEM lane quarter 0 only). Slice 0 opens its idle ring as
            // receive buffers ([slice - 1][half][chunk] 4 KB images), each other slice copies its
            // swizzled partial chunks there with shared::cluster bulk copies completing on slice
            // 0's barrier, and slice 0 adds them in slice order: no global round trips or flags.
            if (dsm > 1 && rbase >= M) {
                // a lane quarter without rows: nothing to exchange or store
            } else if (dsm > 1 && kb0 > 0) {
                const int sl = gid % dsm, nmine = (BN / 32 - half + 1) / 2;
                int i = 0;
#pragma unroll 1
                for (int c = half; c < BN / 32; c += 2, ++i) {
                    uint32_t v[32];
                    tmem_ld32(t_row + uint32_t(c * 32), v);
                    tmem_wait_ld();
                    float4* s4 = reinterpret_cast<float4*>(stg + i * 1024 + lane * 32);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        s4[j ^ (lane & 7)] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                         __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    mbar_wait_cluster(&gobar[ew], 0);
                    const float* rb = reinterpret_cast<const float*>(smem) + size_t((sl - 1) * 2 + half) * nmine * 1024;
                    const uint32_t bar = peer_addr(&ebar[ew], 0);
                    for (int k = 0; k < nmine; ++k) bulk_s2cluster(peer_addr(rb + k * 1024, 0), stg + k * 1024, 4096, bar);
                    mbar_wait_cluster(&donebar[ew], 0);  // slice 0 holds the partial: this CTA may exit
                }
                __syncwarp();
                TRACE2(3);
            } else if (kb0 > 0 && last_seg) {
                // non-head piece, ring idle: TMEM -> swizzled smem -> one 4 KB bulk store per chunk
                int i = 0;
#pragma unroll 1
                for (int c = half; c < BN / 32; c += 2, ++i) {
                    uint32_t v[32];
                    tmem_ld32(t_row + uint32_t(c * 32), v);
                    tmem_wait_ld();
                    float4* s4 = reinterpret_cast<float4*>(stg + i * 1024 + lane * 32);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        s4[j ^ (lane & 7)] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                         __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    float* base = part + (size_t(gid) * CG + rank) * (128 * BN);
                    i = 0;
                    for (int c = half; c < BN / 32; c += 2, ++i)
                        bulk_store_s2g(base + (size_t(c) * 128 + q * 32) * 32, stg + i * 1024, 4096);
                    bulk_commit_wait_all();
                    fence_proxy_async_global();
                    __threadfence();
                    st_release_gpu(&flags[(size_t(gid) * 2 + rank) * 8 + ew], epoch);
                }
                __syncwarp();
                TRACE2(3);
            } else if (kb0 > 0) {
                // non-head piece of a split tile: publish the partial accumulator (the
                // swizzled staging image, copied out linearly: coalesced 512 B per step)
                uint4* dst = reinterpret_cast<uint4*>(part + (size_t(gid) * CG + rank) * (128 * BN) + (q * 32) * 32);
#pragma unroll 1
                for (int c = half; c < BN / 32; c += 2) {
                    uint32_t v[32];
                    tmem_ld32(t_row + uint32_t(c * 32), v);
                    tmem_wait_ld();
                    stage_rows(ep, v, lane);
                    __syncwarp();
                    uint4* d = dst + size_t(c) * 128 * 8;
#pragma unroll
                    for (int j = 0; j < 8; ++j) d[j * 32 + lane] = ep[j * 32 + lane];
                    __syncwarp();
                }
                __threadfence();
                __syncwarp();
                if (lane == 0) st_release_gpu(&flags[(size_t(gid) * 2 + rank) * 8 + ew], epoch);
                TRACE2(3);
            } else {
                // head or whole tile: add the other groups' pieces in group order
                // (groups gid + P, gid + 2P, ... hold them: the same member of the
                // following super-groups)
                int g_last = gid;  // last group holding a piece of this tile
                if (dsm > 1) {
                    // slice 0 of a cluster split (see above): every MMA of this CTA has retired,
                    // so the ring is free for the other slices' partials
                    const int nmine = (BN / 32 - half + 1) / 2;
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&ebar[ew], uint32_t((dsm - 1) * nmine) * 4096u);
                        for (int r = 1; r < dsm; ++r) mbar_arrive_cluster(peer_addr(&gobar[ew], uint32_t(r)));
                    }
                    mbar_wait(&ebar[ew], eph);
                    eph ^= 1;
                    TRACE2(4);
                    if (lane == 0)
                        for (int r = 1; r < dsm; ++r) mbar_arrive_cluster(peer_addr(&donebar[ew], uint32_t(r)));
#pragma unroll 1
                    for (int sl = 1; sl < dsm; ++sl) {
                        const float* rb = reinterpret_cast<const float*>(smem) + size_t((sl - 1) * 2 + half) * nmine * 1024;
                        int i = 0;
#pragma unroll 1
                        for (int c = half; c < BN / 32; c += 2, ++i) {
                            uint32_t v[32];
                            tmem_ld32(t_row + uint32_t(c * 32), v);
                            tmem_wait_ld();
                            const float4* s4 = reinterpret_cast<const float4*>(rb + i * 1024 + lane * 32);
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const float4 a = s4[j ^ (lane & 7)];
                                v[4 * j + 0] = __float_as_uint(__uint_as_float(v[4 * j + 0]) + a.x);
                                v[4 * j + 1] = __float_as_uint(__uint_as_float(v[4 * j + 1]) + a.y);
                                v[4 * j + 2] = __float_as_uint(__uint_as_float(v[4 * j + 2]) + a.z);
                                v[4 * j + 3] = __float_as_uint(__uint_as_float(v[4 * j + 3]) + a.w);
                            }
                            tmem_st32(t_row + uint32_t(c * 32), v);
                        }
                        tmem_wait_st();
                    }
                    __syncwarp();
                    // the two warps of this TMEM quarter swap chunk sets in the epilogue
                    TRACE2(5);
                    tc_fence_before();
                    named_bar(1 + q, 64);
                    tc_fence_after();
                    TRACE2(6);
                } else if (kb1 < num_kb) {
                    if (sk_mode == 2) {
                        g_last = gid + sk_slices - 1;
                    } else {
                        const long tile_end = long(t / P + 1) * num_kb;
                        const int Gs = G / P;
                        int s_last = gid / P;
                        while (s_last + 1 < Gs && sk_start(s_last + 1, Gs, total) < tile_end) ++s_last;
                        g_last = s_last * P + gid % P;
                    }
                }
                for (int g = gid + P; g <= g_last; g += P) {
                    const uint32_t* f = &flags[(size_t(g) * 2 + rank) * 8 + ew];
                    uint32_t spins = 0;
                    while (ld_acquire_gpu(f) != epoch)
                        if (++spins == (1u << 28)) __trap();
                }
                TRACE2(1);
                if (g_last > gid && last_seg) {
                    // ring idle: bulk-load each piece's chunks (fixed group order) and
                    // accumulate into TMEM; the epilogue below then reads final sums
                    const int nmine = (BN / 32 - half + 1) / 2;
                    for (int g = gid + P; g <= g_last; g += P) {
                        if (lane == 0) {
                            fence_proxy_async_global();
                            const float* base = part + (size_t(g) * CG + rank) * (128 * BN);
                            mbar_arrive_expect_tx(&ebar[ew], uint32_t(nmine) * 4096u);
                            int i = 0;
                            for (int c = half; c < BN / 32; c += 2, ++i)
                                bulk_load(stg + i * 1024, base + (size_t(c) * 128 + q * 32) * 32, 4096, &ebar[ew]);
                        }
                        mbar_wait(&ebar[ew], eph);
                        if (g == gid + P) TRACE2(4);
                        eph ^= 1;
                        int i = 0;
#pragma unroll 1
                        for (int c = half; c < BN / 32; c += 2, ++i) {
                            uint32_t v[32];
                            tmem_ld32(t_row + uint32_t(c * 32), v);
                            tmem_wait_ld();
                            const float4* s4 = reinterpret_cast<const float4*>(stg + i * 1024 + lane * 32);
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const float4 a = s4[j ^ (lane & 7)];
                                v[4 * j + 0] = __float_as_uint(__uint_as_float(v[4 * j + 0]) + a.x);
                                v[4 * j + 1] = __float_as_uint(__uint_as_float(v[4 * j + 1]) + a.y);
                                v[4 * j + 2] = __float_as_uint(__uint_as_float(v[4 * j + 2]) + a.z);
                                v[4 * j + 3] = __float_as_uint(__uint_as_float(v[4 * j + 3]) + a.w);
                            }
                            tmem_st32(t_row + uint32_t(c * 32), v);
                        }
                        tmem_wait_st();
                        __syncwarp();  // every lane done with stg before the next piece lands
                    }
                    // the two warps of this TMEM quarter swap chunk sets in the epilogue
                    TRACE2(5);
                    tc_fence_before();
                    named_bar(1 + q, 64);
                    tc_fence_after();
                    TRACE2(6);
                    g_last = gid;
                }
                // pieces of other groups not staged above (tile not in the last segment):
                // coalesced copy of each piece's chunk into ep, then added per row
                auto add_pieces = [&](uint32_t (&v)[32], int c) {
                    for (int g = gid + P; g <= g_last; g += P) {
                        const uint4* src = reinterpret_cast<const uint4*>(part + (size_t(g) * CG + rank) * (128 * BN) +
                                                                          (size_t(c) * 128 + q * 32) * 32);
#pragma unroll
                        for (int j = 0; j < 8; ++j) ep[j * 32 + lane] = __ldcg(src + j * 32 + lane);
                        __syncwarp();
                        add_rows(v, ep, lane);
                        __syncwarp();
                    }
                };
                if constexpr (EPI == EPI_QKV) {
                    // chunk pairs (c, c + 1), c even, hold the rotate-half partners i, i + hd/2 of
                    // one head (Wqkv stores each head's 32-row chunks as [0, 2, 1, 3] for hd = 128)
                    const int64_t blk = q_slot / ea.bs, off = q_slot % ea.bs;
#pragma unroll 1
                    for (int pi = half; pi < BN / 64; pi += 2) {
                        const int c = 2 * pi;
                        uint32_t x1[32], x2[32];
                        tmem_ld32(t_row + uint32_t(c * 32), x1);
                        tmem_ld32(t_row + uint32_t((c + 1) * 32), x2);
                        tmem_wait_ld();
                        if (pi < half + 4) TRACE2(7 + 3 * ((pi - half) >> 1));
                        add_pieces(x1, c);
                        add_pieces(x2, c + 1);
                        const int col = n0 + c * 32;
                        if (col >= N) continue;  // warp-uniform
                        const int hh = col / ea.hd, i0 = (col % ea.hd) / 2;  // i0 < hd/2
                        // this row's packed bf16 result, staged as [lo 64 B | hi 64 B] (lo = columns
                        // i0.., hi = i0 + hd/2..), four 16-byte chunks at a time
                        const bool rot = hh < ea.nq + ea.nkv;  // q or k head: rotate (warp-uniform)
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
                            uint32_t lo[4], hi[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const int j = 4 * jj + k;
                                const float a0 = __uint_as_float(x1[2 * j]) * rs, a1 = __uint_as_float(x1[2 * j + 1]) * rs;
                                const float b0 = __uint_as_float(x2[2 * j]) * rs, b1 = __uint_as_float(x2[2 * j + 1]) * rs;
                                if (rot) {
                                    const float4 f = rc[j];
                                    lo[k] = pack_bf16(a0 * f.x - b0 * f.y, a1 * f.z - b1 * f.w);
                                    hi[k] = pack_bf16(b0 * f.x + a0 * f.y, b1 * f.z + a1 * f.w);
                                } else {
                                    lo[k] = pack_bf16(a0, a1);
                                    hi[k] = pack_bf16(b0, b1);
                                }
                            }
                            ep[lane * 8 + (jj ^ (lane & 7))] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                            ep[lane * 8 + ((jj + 4) ^ (lane & 7))] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                        }
                        // q: this row's head vector (+ i0); k / v: the page of (block, head), whose
                        // row `off` is stored pre-swizzled (kv_page_elem)
                        const bool is_q = hh < ea.nq;  // warp-uniform
                        __nv_bfloat16* dst = nullptr;
                        if (row < M) {
                            if (is_q) dst = ea.q_out + (size_t(row) * ea.nq + hh) * ea.hd + i0;
                            else if (hh < ea.nq + ea.nkv) dst = ea.kc + (size_t(blk) * ea.nkv + (hh - ea.nq)) * ea.bs * ea.hd;
                            else dst = ea.vc + (size_t(blk) * ea.nkv + (hh - ea.nq - ea.nkv)) * ea.bs * ea.hd;
                        }
                        // chunk k < 4 -> column i0 + 8k, else i0 + hd/2 + 8(k-4)
                        __syncwarp();
                        if (pi < half + 4) TRACE2(8 + 3 * ((pi - half) >> 1));
                        const uint64_t dp = reinterpret_cast<uint64_t>(dst);
                        const int colofs = cch < 4 ? cch * 8 : ea.hd / 2 + (cch - 4) * 8;
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int r = 4 * j + crow;
                            const uint64_t d = (uint64_t(__shfl_sync(0xffffffffu, uint32_t(dp >> 32), r)) << 32) |
                                               __shfl_sync(0xffffffffu, uint32_t(dp), r);
                            const int roff = __shfl_sync(0xffffffffu, int(off), r);
                            if (d) {
                                __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(d) +
                                                   (is_q ? colofs : kv_page_elem(roff, i0 + colofs));
                                *reinterpret_cast<uint4*>(p) = ep[r * 8 + (cch ^ (r & 7))];
                            }
                        }
                        __syncwarp();
                        if (pi < half + 4) TRACE2(9 + 3 * ((pi - half) >> 1));
                    }
                } else {
                    // chunks of this warp: c = half, half + 2, ... (SwiGLU: gate/up pairs
                    // (c, c + 1) with c = 2 * half, 2 * half + 4, ...)
                    constexpr int kStep = EPI == EPI_SWIGLU ? 4 : 2;
#pragma unroll
                    for (int i = 0; i < (BN / 32 + kStep - 1) / kStep; ++i) {  // unrolled: xin stays in registers
                        const int c = (EPI == EPI_SWIGLU ? 2 * half : half) + kStep * i;
                        if (c >= BN / 32) break;
                        uint32_t v[32];
                        if constexpr (EPI == EPI_SWIGLU) {
                            uint32_t ut[32];
                            tmem_ld32(t_row + uint32_t(c * 32), v);
                            tmem_ld32(t_row + uint32_t((c + 1) * 32), ut);
                            tmem_wait_ld();
                            add_pieces(v, c);
                            add_pieces(ut, c + 1);
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                v[j] = __float_as_uint(silu(__uint_as_float(v[j]) * rs) * (__uint_as_float(ut[j]) * rs));
                        } else {
                            tmem_ld32(t_row + uint32_t(c * 32), v);
                            tmem_wait_ld();
                            if (i == 0) TRACE2(7);
                            add_pieces(v, c);
                            if (ea.ssq_in) {
#pragma unroll
                                for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * rs);
                            }
                        }
                        stage_rows(ep, v, lane);
                        __syncwarp();
                        if (i == 0) TRACE2(8);
                        const int col = n0 + c * 32;
                        if (col < N) {  // warp-uniform
                            const int ccol = (EPI == EPI_SWIGLU ? col / 2 : col) + cch * 4;
                            float ss[8];
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const int r = 4 * j + crow, grow = rbase + r;
                                const uint4 u = ep[r * 8 + (cch ^ (r & 7))];
                                float4 d = make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z),
                                                       __uint_as_float(u.w));
                                if constexpr (EPI == EPI_RESADD) {
                                    const float4 x0 = xin[i & 1][j];
                                    d.x += x0.x;
                                    d.y += x0.y;
                                    d.z += x0.z;
                                    d.w += x0.w;
                                    ss[j] = d.x * d.x + d.y * d.y + d.z * d.z + d.w * d.w;
                                    if (grow < M) {
                                        *reinterpret_cast<float4*>(static_cast<float*>(out) + size_t(grow) * ldo + ccol) = d;
                                        if (ea.xb_out)
                                            *reinterpret_cast<uint2*>(ea.xb_out + size_t(grow) * ldo + ccol) =
                                                make_uint2(pack_bf16(d.x, d.y), pack_bf16(d.z, d.w));
                                    }
                                } else if (grow < M) {
                                    if constexpr (EPI == EPI_F32) {
                                        *reinterpret_cast<float4*>(static_cast<float*>(out) + size_t(grow) * ldo + ccol) = d;
                                    } else {  // EPI_BF16, EPI_SWIGLU
                                        const uint2 pk = make_uint2(pack_bf16(d.x, d.y), pack_bf16(d.z, d.w));
                                        __nv_bfloat16* dp = static_cast<__nv_bfloat16*>(out) + size_t(grow) * ldo + ccol;
                                        if constexpr (EPI == EPI_BF16) {
                                            if (ea.push_n) {  // TP push reduce-scatter: into the owner's landing zone
                                                const int64_t e = int64_t(grow) * ldo + ccol, u = e >> 3;
                                                const int o = int(u / ea.push_share);
                                                dp = ea.push[o] + ((int64_t(ea.push_rank) * ea.push_share + (u - o * ea.push_share)) << 3) +
                                                     (e & 7);
                                            }
                                        }
                                        *reinterpret_cast<uint2*>(dp) = pk;
                                    }
                                }
                            }
                            if (i == 0) TRACE2(9);
                            if constexpr (EPI == EPI_RESADD) {
                                if (ea.xb_out) {
                                    // per-(row, 32-column chunk) sums of squares: each row's 8 lanes
                                    // reduce in a fixed butterfly order, the 8 rows' chains interleaved
#pragma unroll
                                    for (int m = 1; m <= 4; m <<= 1)
#pragma unroll
                                        for (int j = 0; j < 8; ++j) ss[j] += __shfl_xor_sync(0xffffffffu, ss[j], m);
                                    if (cch == 0) {
#pragma unroll
                                        for (int j = 0; j < 8; ++j) {
                                            const int grow = rbase + 4 * j + crow;
                                            if (grow < M) ea.ssq_out[size_t(grow) * (ldo / 32) + col / 32] = ss[j];
                                        }
                                    }
                                }
                                if (i < 4) TRACE2(10 + i);
                                // refill the used residual slot with chunk i + 2's (overlaps chunk i + 1)
                                const int col2 = col + 4 * 32 + cch * 4;
                                if (c + 4 < BN / 32 && col2 < N) {
#pragma unroll
                                    for (int j = 0; j < 8; ++j) {
                                        const int r = rbase + 4 * j + crow;
                                        if (r < M)  // volatile: issued now, consumed two chunks later
                                            asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                                                         : "=f"(xin[i & 1][j].x), "=f"(xin[i & 1][j].y), "=f"(xin[i & 1][j].z),
                                                           "=f"(xin[i & 1][j].w)
                                                         : "l"(static_cast<const float*>(out) + size_t(r) * ldo + col2));
                                    }
                                }
                            }
                        }
                        __syncwarp();
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            TRACE2(2);
            if (lane == 0) mbar_arrive_cluster_relaxed(CG == 1 ? smem_u32(&tempty[acc]) : tempty_leader + uint32_t(acc * 8));
            if (++acc == 2) {
                acc = 0;
                acc_ph ^= 1;
            }
        }
    }
    if constexpr (EPI == EPI_BF16) {
        // push reduce-scatter: this thread's peer-memory stores performed at system scope
        // before the grid completes (the next kernel's barrier then releases them to the owners)
        if (ea.push_n && warp >= 4) __threadfence_system();
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync();
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_cg<CG>(tmem_base, Cfg::TMEM_COLS);
    }
    if (threadIdx.x == 0) TRACE(7);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// Per-device launch state of one kernel instantiation: the smem attribute is set and the
// co-resident cluster count measured once per device.
constexpr int kMaxDevices = 64;
struct DevOnce {
    bool attr[kMaxDevices] = {};
    int resident[kMaxDevices] = {};
    int clusters[kMaxDevices][9] = {};  // co-resident clusters of s CTAs (dsm), 0 = not measured
};

template <int CG, int BN, int EPI, int AR = 128, int MC = 1>
cudaError_t launch_t(const GemmPlan& p, cudaStream_t st) {
    using Cfg = GemmCfg<CG, BN, AR>;
    static DevOnce once;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    auto kern = gemm_tcgen05_kernel<CG, BN, EPI, AR, MC>;
    if (!once.attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        if (e != cudaSuccess) return e;
        once.attr[dev] = true;
    }
    const int num_mt = (p.M + Cfg::TILE_M - 1) / Cfg::TILE_M;
    const int num_n = (p.N + BN - 1) / BN;
    const int tiles = num_mt * num_n;
    const long iters = long(tiles) * ((p.K + BK - 1) / BK);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG * MC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    // Groups that can be co-resident: stream-K heads spin on other groups, so the
    // grid must never exceed one resident wave. (MC = 2: whole clusters of two pairs.)
    if (once.resident[dev] == 0) {
        const int cs = CG * MC;
        cfg.gridDim = dim3(cs * (p.num_sms / cs));
        int n = 0, r;
        if (CG > 1 && cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) r = n * MC;
        else r = (p.num_sms / cs) * MC;
        once.resident[dev] = r > p.num_sms / CG ? p.num_sms / CG : r;
    }
    int resident = once.resident[dev];
    if (p.max_groups > 0 && p.max_groups < resident) resident = p.max_groups;
    if (MC == 2) resident &= ~1;
    int mode = p.sk_mode, S = p.splits < 1 ? 1 : p.splits;
    if (mode < 0) mode = S > 1 ? 2 : 0;
    if (p.force_sk >= 0) mode = p.force_sk;
    if (p.force_splits > 0) S = p.force_splits;
    if (mode == 3 && num_mt > resident) mode = 0;
    const int rem = tiles % resident;  // tiles of the ragged last wave
    if (mode == 2 && rem > 0 && long(rem) * S > resident) S = resident / rem;
    if (mode == 2 && (S < 2 || rem == 0)) mode = 0;  // nothing to split
    int groups = resident;
    if (mode == 0 && tiles < groups && !(p.epi == EPI_QKV && p.ea.pf_n > 0)) groups = tiles;
    if (mode == 1 && iters < groups) groups = int(iters);
    if (mode == 2 && tiles < resident) groups = tiles * S;
    if (mode == 3) {  // whole super-groups (one member per M-tile), each with >= 1 k-block
        long gs = resident / num_mt;
        if (gs > long(num_n) * ((p.K + BK - 1) / BK)) gs = long(num_n) * ((p.K + BK - 1) / BK);
        groups = int(gs) * num_mt;
    }
    // MC = 2 needs both pairs of a cluster on identical weight k-block sequences: whole
    // tiles or M-lockstep stream-K over an even M-tile count, an even number of pairs
    if (MC == 2 && ((mode != 0 && mode != 3) || (num_mt & 1) || (groups & 1))) return cudaErrorInvalidConfiguration;
    cfg.gridDim = dim3(CG * groups);
    // Split-K over thread-block clusters (dsm): single-CTA tiles of a decode-sized batch (all
    // rows in one TMEM lane quarter), every tile split (one wave), the S slices of a tile one
    // cluster — the partials move through distributed shared memory instead of global memory
    // and flags. Only when all the clusters are co-resident (they run one wave).
    int dsm = 0;
    if (CG == 1 && MC == 1 && p.dsm && mode == 2 && groups == tiles * S && S >= 2 && S <= 8 && p.M <= 32 &&
        (S - 1) * 2 * ((BN / 32 + 1) / 2) * 4096 <= Cfg::STAGES * Cfg::STAGE_BYTES) {
        int& nc = once.clusters[dev][S];
        if (nc == 0) {
            cudaLaunchConfig_t c2 = cfg;
            cudaLaunchAttribute a2[1];
            a2[0].id = cudaLaunchAttributeClusterDimension;
            a2[0].val.clusterDim.x = unsigned(S);
            a2[0].val.clusterDim.y = 1;
            a2[0].val.clusterDim.z = 1;
            c2.attrs = a2;
            c2.numAttrs = 1;
            c2.gridDim = dim3(S * (p.num_sms / S));
            if (cudaOccupancyMaxActiveClusters(&nc, kern, &c2) != cudaSuccess || nc <= 0) {
                cudaGetLastError();
                nc = -1;
            }
        }
        if (nc >= tiles) {
            dsm = S;
            attr[0].val.clusterDim.x = unsigned(S);
        }
    }
    if (p.debug)
        fprintf(stderr, "gemm cg=%d bn=%d mc=%d epi=%d M=%d N=%d K=%d tiles=%d resident=%d mode=%d groups=%d dsm=%d\n",
                CG, BN, MC, EPI, p.M, p.N, p.K, tiles, resident, mode, groups, dsm);
    return cudaLaunchKernelEx(&cfg, kern, p.tmA, p.tmB, p.M, p.row0, p.N, p.K, p.out, p.ldo, num_mt, tiles, p.part,
                              p.flags, p.epoch, mode, S, dsm, p.ea);
}

// Tile shapes compiled: CG=2 pairs with BN in steps of 32, CG=1 with 128 / 256.
constexpr int kBn2[] = {64, 96, 128, 160, 192, 224, 256};

// ============================================================== fused projection chain
// (see ChainPlan in kernels.cuh). CTA pairs, 256 x 256 tiles, the same warp roles,
// operand ring and TMEM double buffer as gemm_tcgen05_kernel<2, 256, *>.

__device__ __forceinline__ uint32_t atom_add_acqrel_gpu(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
// Bounded spin on a flag written by another CTA of this grid (a dependency of an earlier
// work item, which every pair reaches in order: see the deadlock-freedom note below).
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Pollers back off exponentially (64 ns .. 1 us): thousands of threads polling the few lines
// that hold a phase's flags would saturate their L2 slice and slow every epilogue whose
// stores land there.
__device__ __forceinline__ void spin_flag(const uint32_t* f, uint32_t want) {
    if (ld_acquire_gpu(f) == want) return;
    const uint64_t t0 = globaltimer_ns();
    uint32_t ns = 64;
    while (ld_acquire_gpu(f) != want) {  // a schedule bug traps after 2 s instead of hanging the GPU
        __nanosleep(ns);
        if (ns < 1024) ns *= 2;
        if (globaltimer_ns() - t0 > 2000000000ull) __trap();
    }
}
// Wait on n flags (one polling lane), then a warp-wide acquire point.
__device__ __forceinline__ void warp_wait_flags(const uint32_t* f, int n, uint32_t want, int lane) {
    if (lane == 0)
        for (int i = 0; i < n; ++i) spin_flag(f + i, want);
    __syncwarp();
    __threadfence();
}

struct ChainItem {
    int p, m, n, s, kb0, kb1;
};
// The k-th (0..3) of the four 32-column chunks an epilogue warp owns in a 256-column tile, the
// same set the store epilogues walk: RESADD / BF16 every second chunk from `half`; SwiGLU
// gate/up pairs (c, c + 1); QKV rotate-half pairs (c, c + hd / 64). A K-split warp publishes and
// later reduces exactly these chunks.
__device__ __forceinline__ int warp_chunk(int epi, int hd, int half, int k) {
    if (epi == EPI_SWIGLU) return 2 * half + 4 * (k >> 1) + (k & 1);
    if (epi == EPI_QKV) return 2 * (half + 2 * (k >> 1)) + (k & 1);  // rotate-half pairs (c, c + 1)
    return half + 2 * k;
}
__device__ __forceinline__ ChainItem chain_item(const ChainPlan& P, int i) {
    int p = 0;
    while (p + 1 < P.n_phases && i >= P.ph[p + 1].item0) ++p;
    const ChainPhase& ph = P.ph[p];
    const int j = i - ph.item0, S = ph.splits;
    ChainItem it;
    it.p = p;
    it.m = j % P.num_mt;
    const int r = j / P.num_mt;
    it.s = r % S;
    it.n = r / S;
    const int nkb = (ph.K + BK - 1) / BK;
    it.kb0 = it.s * nkb / S;
    it.kb1 = (it.s + 1) * nkb / S;
    return it;
}

// Deadlock freedom: every pair walks its items in increasing global index; an item's
// producer and epilogue wait only on flags of items of EARLIER phases (lower indices), and
// K splits never wait on each other (the last arriver reduces). The lowest unfinished item
// therefore always has its inputs and its pair free to run it. All pairs are co-resident
// (the grid is one resident wave, checked at launch).
// CG = 2: CTA pairs, 256 x 256 tiles (M > 128). CG = 1: single CTAs, 128 x 256 tiles whose A
// stages hold AR rows (decode-sized batches: the projections stream weights, one CTA per SM).
template <int CG, int AR>
__global__ void __launch_bounds__(kThreads, 1) gemm_chain_kernel(const __grid_constant__ ChainPlan P) {
    constexpr int BN = 256;
    using Cfg = GemmCfg<CG, BN, AR>;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2 + 8);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0;
    const bool leader = rank == 0;
    const int gid = blockIdx.x / CG, G = gridDim.x / CG;
    const int M = P.M, num_mt = P.num_mt, total = P.total_items;
    constexpr uint32_t kStageTx = CG * Cfg::STAGE_BYTES;  // bytes a stage's full barrier expects

    if (threadIdx.x == 0) {
        for (int p = 0; p < P.n_phases; ++p) {
            tma_prefetch(&P.tmA[p]);
            tma_prefetch(&P.tmB[p]);
        }
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8 * CG);
        }
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc_cg<CG>(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_launch_dependents();

    // one stage's B (weights) / A (activations) tile, completing on the (pair leader's) full barrier
    auto load_b = [&](int st, const CUtensorMap* tB, int kb, int n0, uint32_t full_leader, uint64_t pol) {
        if constexpr (CG == 1)
            tma_load_2d_hint(sB + st * Cfg::B_BYTES, tB, kb * BK, n0, &full[st], pol);
        else
            tma_load_2d_cg2_hint(sB + st * Cfg::B_BYTES, tB, kb * BK, n0, full_leader + uint32_t(st * 8), pol);
    };
    auto load_a = [&](int st, const CUtensorMap* tA, int kb, int m0, uint32_t full_leader, uint64_t pol) {
        if constexpr (CG == 1)
            tma_load_2d_hint(sA + st * Cfg::A_BYTES, tA, kb * BK, m0, &full[st], pol);
        else
            tma_load_2d_cg2_hint(sA + st * Cfg::A_BYTES, tA, kb * BK, m0, full_leader + uint32_t(st * 8), pol);
    };

    if (warp == 0) {  // ---------------- TMA producer (both CTAs; lane 0 issues, the warp checks flags)
        const uint32_t full_leader = CG == 2 ? peer_addr(full, 0) : 0;
        const uint64_t polA = l2_policy_evict_last();
        const uint64_t polB = l2_policy_evict_first();
        // the first item's first weight stages before the grid-dependency wait
        int npre = 0;
        if (gid < total) {
            const ChainItem it = chain_item(P, gid);
            const int n0 = it.n * BN + Cfg::B_ROWS * int(rank);
            npre = it.kb1 - it.kb0 < STAGES ? it.kb1 - it.kb0 : STAGES;
            if (lane == 0)
                for (int j = 0; j < npre; ++j) {
                    if (leader) mbar_arrive_expect_tx(&full[j], kStageTx);
                    load_b(j, &P.tmB[it.p], it.kb0 + j, n0, full_leader, polB);
                }
        }
        pdl_wait();
        const uint32_t E = P.epoch + (P.epoch_base ? *reinterpret_cast<const volatile uint32_t*>(P.epoch_base) : 0u);
        // Known-ready prefix of the dependency phase's tiles, per M-tile (lane m holds M-tile
        // m's; more than 32 M-tiles: no cache). Flags only go up within a launch, so a tile
        // seen ready stays ready: most items then need no flag traffic at all.
        int kr = -1, kr_dep = -2;
        int s = 0, itn = 0;
        uint32_t ph = 0;
        for (int i = gid; i < total; i += G) {
            const ChainItem it = chain_item(P, i);
            const ChainPhase& cp = P.ph[it.p];
            if (P.trace && leader && lane == 0) P.trace[size_t(i) * 16 + 0] = globaltimer_ns();
            const int m0 = it.m * Cfg::TILE_M + 128 * int(rank);
            const int n0 = it.n * BN + Cfg::B_ROWS * int(rank);
            const CUtensorMap* tA = &P.tmA[it.p];
            const CUtensorMap* tB = &P.tmB[it.p];
            const uint32_t* rdy = cp.dep >= 0 ? P.ph[cp.dep].ready + size_t(it.m) * P.ph[cp.dep].num_n : nullptr;
            const int dcols = cp.dep >= 0 ? P.ph[cp.dep].out_cols : 1;
            const int nd = cp.dep >= 0 ? P.ph[cp.dep].num_n : 0;
            if (cp.dep != kr_dep) {
                kr = -1;
                kr_dep = cp.dep;
            }
            const bool cache = num_mt <= 32;
            int known = cache ? __shfl_sync(0xffffffffu, kr, it.m & 31) : -1;
            for (int kb = it.kb0; kb < it.kb1; ++kb, ++itn) {
                // the stage's weight tile first: it depends on nothing, so weight streaming
                // runs ahead of the activations' readiness
                if (lane == 0) {
                    const bool pre = itn < npre;
                    if (!pre) {
                        mbar_wait(&empty[s], ph ^ 1);
                        if (leader) mbar_arrive_expect_tx(&full[s], kStageTx);
                        load_b(s, tB, kb, n0, full_leader, polB);
                    }
                }
                if (rdy) {  // the producing phase's output tile covering these 64 columns
                    const int ct = kb * BK / dcols;
                    if (ct > known) {
                        int cnt = 0;
                        for (;;) {  // one round trip checks 32 tiles
                            const int t = ct + lane;
                            const bool ok = t >= nd || ld_acquire_gpu(rdy + t) == E;
                            const unsigned nm = ~__ballot_sync(0xffffffffu, ok);
                            cnt = nm ? __ffs(nm) - 1 : 32;
                            if (cnt > 0) break;
                            if (lane == 0) spin_flag(rdy + ct, E);
                            __syncwarp();
                        }
                        known = ct + cnt - 1;
                        if (cache && lane == (it.m & 31)) kr = known;
                        __syncwarp();
                        if (lane == 0) fence_proxy_async_global();
                    }
                }
                if (lane == 0) load_a(s, tA, kb, m0, full_leader, polA);
                __syncwarp();
                if (++s == STAGES) {
                    s = 0;
                    ph ^= 1;
                }
            }
            if (P.trace && leader && lane == 0) P.trace[size_t(i) * 16 + 1] = globaltimer_ns();
        }
    } else if (warp == 1) {
        if (leader) {  // ---------------- MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(Cfg::TILE_M, BN);
            const uint64_t adesc0 = umma_desc_sw128(smem_u32(sA)), bdesc0 = umma_desc_sw128(smem_u32(sB));
            int s = 0, acc = 0;
            uint32_t ph = 0, acc_ph = 0;
            for (int i = gid; i < total; i += G) {
                const ChainItem it = chain_item(P, i);
                mbar_wait(&tempty[acc], acc_ph ^ 1);
                tc_fence_after();
                if (P.trace && lane == 0) P.trace[size_t(i) * 16 + 2] = globaltimer_ns();
                const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
                const int nk = it.kb1 - it.kb0;
                for (int k = 0; k < nk; ++k) {
                    mbar_wait(&full[s], ph);
                    const uint64_t ad = adesc0 + uint64_t((s * Cfg::A_BYTES) >> 4);
                    const uint64_t bd = bdesc0 + uint64_t((s * Cfg::B_BYTES) >> 4);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk)
                            mma_cg<CG>(d_tmem, ad + uint64_t(2 * kk), bd + uint64_t(2 * kk), idesc,
                                       (k > 0 || kk > 0) ? 1u : 0u);
                        commit_cg<CG>(&empty[s]);
                    }
                    __syncwarp();
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (elect_one()) commit_cg<CG>(&tfull[acc]);
                __syncwarp();
                if (P.trace && lane == 0) P.trace[size_t(i) * 16 + 3] = globaltimer_ns();
                if (++acc == 2) {
                    acc = 0;
                    acc_ph ^= 1;
                }
            }
        }
    } else {  // ---------------------------- epilogue warps 2..9
        pdl_wait();
        const uint32_t E = P.epoch + (P.epoch_base ? *reinterpret_cast<const volatile uint32_t*>(P.epoch_base) : 0u);
        const int q = warp & 3;
        const int ew = warp - 2, half = ew >> 2;
        const uint32_t tempty_leader = CG == 2 ? peer_addr(tempty, 0) : smem_u32(tempty);
        const int trace_ew = M <= 32 ? 2 : 0;  // dev timeline: a warp whose rows hold tokens
        const int rloc = 128 * int(rank) + q * 32 + lane;
        uint4* ep = reinterpret_cast<uint4*>(smem + STAGES * Cfg::STAGE_BYTES + 1024 + ew * 4096);
        const int crow = lane >> 3, cch = lane & 7;
        int acc = 0;
        uint32_t acc_ph = 0;
        auto release_acc = [&]() {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader + uint32_t(acc * 8));
            if (++acc == 2) {
                acc = 0;
                acc_ph ^= 1;
            }
        };
        for (int i = gid; i < total; i += G) {
            const ChainItem it = chain_item(P, i);
            const ChainPhase& cp = P.ph[it.p];
            const EpiArgs& ea = cp.ea;
            const int S = cp.splits, EPI = cp.epi, N = cp.N, ldo = cp.ldo;
            const int tile = it.m * cp.num_n + it.n;
            const int m0 = it.m * Cfg::TILE_M, n0 = it.n * BN;
            const int row = m0 + rloc, rbase = row - lane;
            const bool live = rbase < M;  // warp-uniform: this warp's 32 rows hold tokens
            // inputs written by earlier items: acquire their tiles' flags, then read coherently
            if (ea.ssq_in && cp.dep >= 0)
                warp_wait_flags(P.ph[cp.dep].ready + size_t(it.m) * P.ph[cp.dep].num_n, P.ph[cp.dep].num_n, E, lane);
            if (cp.res_dep >= 0) warp_wait_flags(P.ph[cp.res_dep].ready + tile, 1, E, lane);
            float rs = 1.f;
            if (ea.ssq_in) {  // folded RMSNorm row scale (coalesced loads + transpose-reduce)
                const int n4 = ea.ssq_in_n >> 2;
                float a[32];
#pragma unroll
                for (int r = 0; r < 32; ++r) a[r] = 0.f;
                for (int k = lane; k - lane < n4; k += 32) {
#pragma unroll
                    for (int r = 0; r < 32; ++r) {
                        if (k < n4 && rbase + r < M) {
                            const float4 w = __ldcg(reinterpret_cast<const float4*>(ea.ssq_in + size_t(rbase + r) * ea.ssq_in_n) + k);
                            a[r] += (w.x + w.y) + (w.z + w.w);
                        }
                    }
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    const bool up = lane & off;
#pragma unroll
                    for (int k = 0; k < off; ++k) {
                        const float send = up ? a[k] : a[k + off];
                        const float keep = up ? a[k + off] : a[k];
                        a[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                    }
                }
                rs = rsqrtf(a[0] * ea.inv_dim + ea.eps);
            }
            // QKV: position / slot of this row (batch inputs); the RoPE factors are read at use
            // (L1-resident table rows; preloading them spilled registers)
            int q_pos = 0;
            int64_t q_slot = 0;
            if (EPI == EPI_QKV && row < M) {
                q_pos = ea.pos[row];
                q_slot = ea.slot[row];
            }
            mbar_wait(&tfull[acc], acc_ph);
            tc_fence_after();
            if (P.trace && leader && ew == trace_ew && lane == 0) P.trace[size_t(i) * 16 + 4] = globaltimer_ns();
            const uint32_t t_row = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
            bool from_part = false;
            if (S > 1) {
                // publish this split's partial (staged swizzled image, copied out coalesced)
                uint4* dst = reinterpret_cast<uint4*>(cp.part + (((size_t(tile) * S + it.s) * CG + rank) * 8) * 4096 +
                                                      (q * 32) * 32);
#pragma unroll 1
                for (int k = 0; k < BN / 64 && live; ++k) {
                    const int c = warp_chunk(EPI, ea.hd, half, k);
                    uint32_t v[32];
                    tmem_ld32(t_row + uint32_t(c * 32), v);
                    tmem_wait_ld();
                    stage_rows(ep, v, lane);
                    __syncwarp();
                    uint4* d = dst + size_t(c) * 128 * 8;
#pragma unroll
                    for (int j = 0; j < 8; ++j) d[j * 32 + lane] = ep[j * 32 + lane];
                    __syncwarp();
                }
                release_acc();
                __threadfence();
                __syncwarp();
                if (P.trace && leader && ew == trace_ew && lane == 0) P.trace[size_t(i) * 16 + 12] = globaltimer_ns();
                uint32_t old = 0;
                if (lane == 0) old = atom_add_acqrel_gpu(&cp.pcnt[(size_t(tile) * 2 + rank) * 8 + ew], 1u);
                old = __shfl_sync(0xffffffffu, old, 0);
                if (old != uint32_t(S - 1)) continue;  // another split finishes this slice
                if (lane == 0) cp.pcnt[(size_t(tile) * 2 + rank) * 8 + ew] = 0u;
                __syncwarp();
                __threadfence();  // every split's partial (acquired by lane 0) before the reads below
                from_part = true;
            }
            // chunk c (32 columns) of this warp's 32 rows: from TMEM, or the sum of every
            // split's partial in split order
            auto load_chunk = [&](int c, uint32_t (&v)[32]) {
                if (!from_part) {
                    tmem_ld32(t_row + uint32_t(c * 32), v);
                    tmem_wait_ld();
                    return;
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = 0u;
                if (CG == 1 && M <= 32) {
                    // only row quarter 0 holds tokens: the idle warps' staging buffers of this
                    // half (4 x 4 KB, contiguous) take four splits' chunks per round trip
                    uint4* stg4 = reinterpret_cast<uint4*>(smem + STAGES * Cfg::STAGE_BYTES + 1024 + (4 * half) * 4096);
                    for (int sp0 = 0; sp0 < S; sp0 += 4) {
                        const int n = S - sp0 < 4 ? S - sp0 : 4;
                        for (int i = 0; i < n; ++i) {
                            const uint4* src = reinterpret_cast<const uint4*>(
                                cp.part + (((size_t(tile) * S + sp0 + i) * CG + rank) * 8) * 4096 + (size_t(c) * 128 + q * 32) * 32);
#pragma unroll
                            for (int j = 0; j < 8; ++j) cp_async16(smem_u32(stg4 + i * 256 + j * 32 + lane), src + j * 32 + lane);
                        }
                        cp_async_commit();
                        cp_async_wait<0>();
                        __syncwarp();
                        for (int i = 0; i < n; ++i) add_rows(v, stg4 + i * 256, lane);  // split order
                        __syncwarp();
                    }
                    return;
                }
                for (int sp = 0; sp < S; ++sp) {  // added in split order (deterministic)
                    const uint4* src = reinterpret_cast<const uint4*>(
                        cp.part + (((size_t(tile) * S + sp) * CG + rank) * 8) * 4096 + (size_t(c) * 128 + q * 32) * 32);
                    // global -> smem without a register round trip (8 x 16 B in flight per lane)
#pragma unroll
                    for (int j = 0; j < 8; ++j) cp_async16(smem_u32(ep + j * 32 + lane), src + j * 32 + lane);
                    cp_async_commit();
                    cp_async_wait<0>();
                    __syncwarp();
                    add_rows(v, ep, lane);
                    __syncwarp();
                }
            };
            if (!live) {
                // no token rows in this warp's quarter of the tile: nothing to store
            } else if (EPI == EPI_QKV) {
                const int64_t blk = q_slot / ea.bs, off = q_slot % ea.bs;
#pragma unroll 1
                for (int pi = half; pi < BN / 64; pi += 2) {  // rotate-half pairs (c, c + 1), c even
                    const int c = 2 * pi;
                    uint32_t x1[32], x2[32];
                    load_chunk(c, x1);
                    load_chunk(c + 1, x2);
                    const int col = n0 + c * 32;
                    if (col >= N) continue;
                    const int hh = col / ea.hd, i0 = (col % ea.hd) / 2;
                    const bool rot = hh < ea.nq + ea.nkv;
                    const float4* cs = reinterpret_cast<const float4*>(ea.rope + size_t(q_pos) * (ea.hd / 2) + i0);
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        uint32_t lo[4], hi[4];
                        float4 rc[4];
                        if (rot) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) rc[k] = __ldg(cs + 4 * jj + k);
                        }
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int j = 4 * jj + k;
                            const float a0 = __uint_as_float(x1[2 * j]) * rs, a1 = __uint_as_float(x1[2 * j + 1]) * rs;
                            const float b0 = __uint_as_float(x2[2 * j]) * rs, b1 = __uint_as_float(x2[2 * j + 1]) * rs;
                            if (rot) {
                                const float4 f = rc[k];
                                lo[k] = pack_bf16(a0 * f.x - b0 * f.y, a1 * f.z - b1 * f.w);
                                hi[k] = pack_bf16(b0 * f.x + a0 * f.y, b1 * f.z + a1 * f.w);
                            } else {
                                lo[k] = pack_bf16(a0, a1);
                                hi[k] = pack_bf16(b0, b1);
                            }
                        }
                        ep[lane * 8 + (jj ^ (lane & 7))] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                        ep[lane * 8 + ((jj + 4) ^ (lane & 7))] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                    }
                    const bool is_q = hh < ea.nq;  // k / v rows go into pre-swizzled pages (kv_page_elem)
                    __nv_bfloat16* dst = nullptr;
                    if (row < M) {
                        if (is_q) dst = ea.q_out + (size_t(row) * ea.nq + hh) * ea.hd + i0;
                        else if (hh < ea.nq + ea.nkv) dst = ea.kc + (size_t(blk) * ea.nkv + (hh - ea.nq)) * ea.bs * ea.hd;
                        else dst = ea.vc + (size_t(blk) * ea.nkv + (hh - ea.nq - ea.nkv)) * ea.bs * ea.hd;
                    }
                    __syncwarp();
                    const uint64_t dp = reinterpret_cast<uint64_t>(dst);
                    const int colofs = cch < 4 ? cch * 8 : ea.hd / 2 + (cch - 4) * 8;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int r = 4 * j + crow;
                        const uint64_t d = (uint64_t(__shfl_sync(0xffffffffu, uint32_t(dp >> 32), r)) << 32) |
                                           __shfl_sync(0xffffffffu, uint32_t(dp), r);
                        const int roff = __shfl_sync(0xffffffffu, int(off), r);
                        if (d) {
                            __nv_bfloat16* pp = reinterpret_cast<__nv_bfloat16*>(d) +
                                                (is_q ? colofs : kv_page_elem(roff, i0 + colofs));
                            *reinterpret_cast<uint4*>(pp) = ep[r * 8 + (cch ^ (r & 7))];
                        }
                    }
                    __syncwarp();
                }
            } else if (EPI == EPI_SWIGLU) {
#pragma unroll 1
                for (int c = 2 * half; c < BN / 32; c += 4) {
                    uint32_t v[32], ut[32];
                    load_chunk(c, v);
                    load_chunk(c + 1, ut);
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        v[j] = __float_as_uint(silu(__uint_as_float(v[j]) * rs) * (__uint_as_float(ut[j]) * rs));
                    stage_rows(ep, v, lane);
                    __syncwarp();
                    const int col = n0 + c * 32;
                    if (col < N) {
                        const int ccol = col / 2 + cch * 4;
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int r = 4 * j + crow, grow = rbase + r;
                            const uint4 u = ep[r * 8 + (cch ^ (r & 7))];
                            if (grow < M)
                                *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(cp.out) + size_t(grow) * ldo + ccol) =
                                    make_uint2(pack_bf16(__uint_as_float(u.x), __uint_as_float(u.y)),
                                               pack_bf16(__uint_as_float(u.z), __uint_as_float(u.w)));
                        }
                    }
                    __syncwarp();
                }
            } else {  // EPI_RESADD (x_f32 += D, + bf16 copy and per-chunk sums of squares) / EPI_BF16
                // residual of chunk c (coalesced layout, rows rbase + 4j + crow), loaded a chunk ahead
                float4 xin[2][8];
                auto load_res = [&](int c, float4 (&xr)[8]) {
                    const int col = n0 + c * 32 + cch * 4;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int grow = rbase + 4 * j + crow;
                        xr[j] = (EPI == EPI_RESADD && grow < M && col < N)
                                    ? __ldcg(reinterpret_cast<const float4*>(static_cast<const float*>(cp.out) + size_t(grow) * ldo + col))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                };
                if (EPI == EPI_RESADD) load_res(half, xin[0]);
#pragma unroll
                for (int ci = 0; ci < BN / 64; ++ci) {
                    const int c = half + 2 * ci;
                    if (EPI == EPI_RESADD && ci + 1 < BN / 64) load_res(c + 2, xin[(ci + 1) & 1]);
                    uint32_t v[32];
                    load_chunk(c, v);
                    if (ea.ssq_in) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * rs);
                    }
                    stage_rows(ep, v, lane);
                    __syncwarp();
                    const int col = n0 + c * 32;
                    if (col < N) {
                        const int ccol = col + cch * 4;
                        float ss[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int r = 4 * j + crow, grow = rbase + r;
                            const uint4 u = ep[r * 8 + (cch ^ (r & 7))];
                            float4 d = make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z),
                                                   __uint_as_float(u.w));
                            ss[j] = 0.f;
                            if (grow < M) {
                                if (EPI == EPI_RESADD) {
                                    float* xp = static_cast<float*>(cp.out) + size_t(grow) * ldo + ccol;
                                    const float4 x0 = xin[ci & 1][j];
                                    d.x += x0.x;
                                    d.y += x0.y;
                                    d.z += x0.z;
                                    d.w += x0.w;
                                    ss[j] = d.x * d.x + d.y * d.y + d.z * d.z + d.w * d.w;
                                    *reinterpret_cast<float4*>(xp) = d;
                                    if (ea.xb_out)
                                        *reinterpret_cast<uint2*>(ea.xb_out + size_t(grow) * ldo + ccol) =
                                            make_uint2(pack_bf16(d.x, d.y), pack_bf16(d.z, d.w));
                                } else {
                                    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(cp.out) + size_t(grow) * ldo + ccol) =
                                        make_uint2(pack_bf16(d.x, d.y), pack_bf16(d.z, d.w));
                                }
                            }
                        }
                        if (EPI == EPI_RESADD && ea.xb_out) {
#pragma unroll
                            for (int mm = 1; mm <= 4; mm <<= 1)
#pragma unroll
                                for (int j = 0; j < 8; ++j) ss[j] += __shfl_xor_sync(0xffffffffu, ss[j], mm);
                            if (cch == 0) {
#pragma unroll
                                for (int j = 0; j < 8; ++j) {
                                    const int grow = rbase + 4 * j + crow;
                                    if (grow < M) ea.ssq_out[size_t(grow) * (ldo / 32) + col / 32] = ss[j];
                                }
                            }
                        }
                    }
                    __syncwarp();
                    if (P.trace && leader && ew == trace_ew && lane == 0) P.trace[size_t(i) * 16 + 6 + ci] = globaltimer_ns();
                }
            }
            if (P.trace && leader && ew == trace_ew && lane == 0) P.trace[size_t(i) * 16 + 14] = globaltimer_ns();
            if (!from_part) release_acc();
            // this warp's share of the tile is stored: count it; the 16th warp publishes the tile
            fence_proxy_async_global();  // consumers read these stores through TMA (async proxy)
            __threadfence();
            __syncwarp();
            if (lane == 0) {
                const uint32_t old = atom_add_acqrel_gpu(&cp.rcnt[tile], 1u);
                if (P.trace && leader && ew == trace_ew) P.trace[size_t(i) * 16 + 15] = globaltimer_ns();
                if (old == uint32_t(CG) * 8u - 1u) {
                    cp.rcnt[tile] = 0u;
                    st_release_gpu(&cp.ready[tile], E);
                    if (P.trace) P.trace[size_t(i) * 16 + 5] = globaltimer_ns();
                }
            }
        }
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync();
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_cg<CG>(tmem_base, Cfg::TMEM_COLS);
    }
}

}  // namespace

void gemm_chain_finalize(ChainPlan& p) {
    int item = 0;
    for (int i = 0; i < p.n_phases; ++i) {
        ChainPhase& ph = p.ph[i];
        ph.num_n = (ph.N + 255) / 256;
        ph.item0 = item;
        item += p.num_mt * ph.num_n * (ph.splits < 1 ? 1 : ph.splits);
    }
    p.total_items = item;
}

namespace {
template <int CG, int AR>
cudaError_t chain_launch_t(const ChainPlan& p, cudaStream_t st) {
    using Cfg = GemmCfg<CG, 256, AR>;
    static DevOnce once;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    auto kern = gemm_chain_kernel<CG, AR>;
    if (!once.attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        if (e != cudaSuccess) return e;
        once.attr[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    // every group must be resident at once (flag waits between groups)
    if (once.resident[dev] == 0) {
        cfg.gridDim = dim3(CG * (p.num_sms / CG));
        int n = 0;
        if (CG == 1 || cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) n = p.num_sms / CG;
        once.resident[dev] = n > p.num_sms / CG ? p.num_sms / CG : n;
    }
    int groups = once.resident[dev];
    if (groups > p.total_items) groups = p.total_items;
    if (groups < 1) return cudaSuccess;
    cfg.gridDim = dim3(CG * groups);
    if (p.debug)
        fprintf(stderr, "gemm chain cg=%d ar=%d M=%d phases=%d items=%d groups=%d\n", CG, AR, p.M, p.n_phases,
                p.total_items, groups);
    return cudaLaunchKernelEx(&cfg, kern, p);
}
}  // namespace

cudaError_t gemm_chain_launch(const ChainPlan& p, cudaStream_t st) {
    if (p.cg == 2) return chain_launch_t<2, 128>(p, st);
    if (p.cg == 1 && p.ar == 32) return chain_launch_t<1, 32>(p, st);
    if (p.cg == 1) return chain_launch_t<1, 128>(p, st);
    return cudaErrorInvalidValue;
}

namespace {
}  // namespace

Tuning tuning_from_env() {
    Tuning t;
    auto geti = [](const char* name, int& v) {
        if (const char* f = getenv(name)) v = atoi(f);
    };
    geti("SS_ATTN_TC_MODE", t.attn_tc_mode);
    geti("SS_ATTN_ORDER", t.attn_order);
    geti("SS_ATTN_L2HINT", t.attn_l2hint);
    geti("SS_ATTN_TC2_FIRST", t.attn_tc2_first);
    geti("SS_ATTN_PF_PAGES", t.attn_pf_pages);
    geti("SS_GEMM_L2HINT", t.gemm_l2hint);
    geti("SS_GEMM_SK", t.gemm_sk);
    geti("SS_GEMM_SPLITS", t.gemm_splits);
    geti("SS_GEMM_BN", t.gemm_bn);
    geti("SS_GEMM_CG", t.gemm_cg);
    if (getenv("SS_GEMM_AR128")) t.gemm_ar128 = 1;
    if (getenv("SS_GEMM_DEBUG")) t.gemm_debug = 1;
    geti("SS_GEMM_LDO_PAD", t.ldo_pad);
    geti("SS_CHAIN", t.chain);
    if (const char* f = getenv("SS_CHAIN_S"))
        sscanf(f, "%d,%d,%d,%d", &t.chain_splits[0], &t.chain_splits[1], &t.chain_splits[2], &t.chain_splits[3]);
    if (getenv("SS_CHAIN_DEBUG")) t.chain_debug = 1;
    geti("SS_CHAIN_TRACE", t.chain_trace);
    geti("SS_GEMM_MAXG", t.gemm_max_groups);
    geti("SS_GEMM_DSM", t.gemm_dsm);
    geti("SS_GEMM_MC", t.gemm_mc);
    static const char* names[5] = {"SS_GEMM_QKV", "SS_GEMM_O", "SS_GEMM_GATEUP", "SS_GEMM_DOWN", "SS_GEMM_LMHEAD"};
    for (int i = 0; i < 5; ++i)
        if (const char* f = getenv(names[i])) {
            int md = -1, bn = 0, sp = 1;
            if (sscanf(f, "%d,%d,%d", &md, &bn, &sp) >= 2) {
                t.gemm_force[i][0] = md;
                t.gemm_force[i][1] = bn;
                t.gemm_force[i][2] = sp;
            }
        }
    return t;
}

bool make_tmap_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                  uint32_t box_cols) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Co-resident thread-block clusters of s single-CTA GEMM CTAs on this device (the dsm split
// needs all of a launch's clusters resident at once): measured once per device and size.
int gemm_dsm_clusters(int s) {
    static int cache[kMaxDevices][9] = {};
    int dev = 0;
    if (s < 2 || s > 8 || cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
    int& nc = cache[dev][s];
    if (nc == 0) {
        using Cfg = GemmCfg<1, 128, 32>;
        auto kern = gemm_tcgen05_kernel<1, 128, EPI_BF16, 32>;
        cudaLaunchConfig_t c = {};
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = unsigned(s);
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        c.attrs = a;
        c.numAttrs = 1;
        c.blockDim = dim3(kGemmThreads);
        c.dynamicSmemBytes = Cfg::SMEM;
        c.gridDim = dim3(s * 16);
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM) != cudaSuccess ||
            cudaOccupancyMaxActiveClusters(&nc, kern, &c) != cudaSuccess || nc <= 0) {
            cudaGetLastError();
            nc = -1;
        }
    }
    return nc;
}

GemmShape gemm_pick(int M, int N, int K, int epi, int num_sms, const Tuning& tu) {
    const int force_bn = tu.gemm_bn, force_cg = tu.gemm_cg, force_s = tu.gemm_splits, force_mode = tu.gemm_sk;
    const bool swiglu = epi == EPI_SWIGLU;
    GemmShape best{M > 128 ? 2 : 1, swiglu ? 256 : 128, 1, -1};
    double best_cost = 1e30;
    // Cost model calibrated inside the Mistral forward (profiles/r01/gemm_class_sweep.txt,
    // scripts/gemm_class_sweep.py): per 64 k-blocks a CTA-pair tile's main loop takes
    // ~15 + 0.0135 * BN us in K-lockstep (L2 -> SM fill bound, so narrow tiles save
    // little), 1.18x that in M-lockstep stream-K (the groups no longer share A
    // k-blocks in L2); every launch pays ~3 + 0.07 * BN us of start-up and exposed
    // last epilogue, stream-K ~6 us more (partial write + fixup of split tiles).
    // Whole tiles go round-robin (mode 0); a ragged last wave can be split in K
    // (mode 2); mode 3 balances every group exactly.
    auto tile_us = [](int c, int b) {
        if (c == 1) return b == 256 ? 28.6 : b == 128 ? 20.4 : 11.0;  // 64: weight streaming, 16 stages
        return 15.0 + 0.0135 * b;
    };
    const double kscale = double((K + BK - 1) / BK) / 64.0;
    auto consider = [&](int cg, int bn) {
        if (swiglu && bn % 64) return;
        if (epi == EPI_QKV && bn % 64) return;  // whole rotate-half chunk pairs per tile
        if (force_bn && bn != force_bn) return;
        if (force_cg && cg != force_cg) return;
        const long num_mt = (M + 128 * cg - 1) / (128 * cg), num_n = (N + bn - 1) / bn;
        const long tiles = num_mt * num_n;
        const long slots = num_sms / cg;
        const long full = tiles / slots, rem = tiles % slots;
        const double t1 = tile_us(cg, bn) * kscale, epi_us = 3.0 + 0.07 * bn;
        if (num_mt <= slots && (force_mode < 0 || force_mode == 3)) {
            const long gs = slots / num_mt, nkb = (K + BK - 1) / BK;
            const long per = (num_n * nkb + gs - 1) / gs;
            // (single-CTA tiles at M <= 128 are weight-streaming bound per SM; their split
            // partials cost ~10 us more than the spread saves unless K is long: decode-only
            // sweep, profiles/r01/gemm_class_sweep.txt)
            const double cost = double(per) / 64.0 * 1.18 * tile_us(cg, bn) + epi_us + 6.0 + (cg == 1 ? 10.0 : 0.0);
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best = GemmShape{cg, bn, 1, 3};
            }
        }
        if (force_mode == 3) return;
        for (int S = 1; S <= 4; ++S) {
            if (force_s && S != force_s) continue;
            if (S > 1 && (rem == 0 || rem * S > slots)) break;
            // split partials of 32-row single-CTA tiles are 4x smaller (decode-only sweep:
            // 2.5 + 2.7 S fits the measured S = 2..4 overheads); through the cluster's shared
            // memory (dsm, when all the tile clusters fit at once) 1.5 + 2.5 S (decode-only
            // step sweep, profiles/r02/ab_gemm_dsm.txt: QKV S = 2 over S = 3 through global
            // memory, O S = 3, down S = 4)
            const bool dsm = cg == 1 && M <= 32 && tu.gemm_dsm && S > 1 && rem == tiles && tiles <= gemm_dsm_clusters(S);
            const double ovh = dsm ? 1.5 + 2.5 * S : cg == 1 && M <= 32 ? 2.5 + 2.7 * S : 8.0 + 2.0 * S;
            const double last = rem == 0 ? 0.0 : t1 / S + (S > 1 ? ovh : 0.0);
            const double cost = double(full) * t1 + last + epi_us;
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best = GemmShape{cg, bn, S, S > 1 ? 2 : 0};
            }
        }
    };
    if (M <= 128 || force_cg == 1) {
        consider(1, 256);
        consider(1, 128);
        // BN = 64 weight-streaming tiles (32-row A stages): only when forced — measured slower
        // on the decode-only step (6.33 vs 6.14 ms, profiles/r02/ab_decode_bn64.txt)
        if (M <= 32 && !tu.gemm_ar128 && force_bn == 64) consider(1, 64);
    }
    best.ar = (best.cg == 1 && M <= 32 && !tu.gemm_ar128) ? 32 : 128;
    if (M > 128 && force_cg != 1)
        for (int bn : kBn2) consider(2, bn);
    return best;
}

int gemm_mc(const GemmShape& s, int M, const Tuning& tu) {
    if (!tu.gemm_mc || s.cg != 2 || (s.mode != 0 && s.mode != 3) || (s.bn != 128 && s.bn != 256)) return 1;
    const int num_mt = (M + 255) / 256;
    return num_mt % 2 == 0 ? 2 : 1;
}

bool gemm_prepare(GemmPlan& p, const void* A, uint64_t a_rows, const void* B, int M, int N, int K, void* out,
                  int ldo, int epi, int num_sms, const Tuning& tu, int bn) {
    if (M < 1 || N < 32 || K < 16 || N % 32 || K % 8 || (epi == EPI_SWIGLU && N % 64) || epi == EPI_QKV) return false;
    p.M = M;
    p.N = N;
    p.K = K;
    p.out = out;
    p.ldo = ldo;
    p.epi = epi;
    p.num_sms = num_sms;
    const GemmShape s = gemm_pick(M, N, K, epi, num_sms, tu);
    p.force_sk = tu.gemm_sk;
    p.force_splits = tu.gemm_splits;
    p.debug = tu.gemm_debug;
    p.max_groups = tu.gemm_max_groups;
    p.dsm = tu.gemm_dsm;
    p.cg = s.cg;
    p.bn = bn ? bn : s.bn;
    p.splits = s.splits;
    p.sk_mode = s.mode;
    p.ar = (p.cg == 1 && p.bn == s.bn) ? s.ar : 128;
    p.mc = p.bn == s.bn ? gemm_mc(s, M, tu) : 1;
    if (!make_tmap_2d(&p.tmA, A, a_rows, uint64_t(K), uint32_t(p.ar), BK)) return false;
    if (!make_tmap_2d(&p.tmB, B, uint64_t(N), uint64_t(K), uint32_t(p.bn / p.cg / p.mc), BK)) return false;
    return true;
}

cudaError_t gemm_launch(const GemmPlan& p, cudaStream_t st) {
    if (p.cg == 2 && p.mc == 2) {
#define SS_GEMM_CASE_MC(BNv)                                                          \
    if (p.bn == BNv) {                                                               \
        if (p.epi == EPI_BF16) return launch_t<2, BNv, EPI_BF16, 128, 2>(p, st);     \
        if (p.epi == EPI_RESADD) return launch_t<2, BNv, EPI_RESADD, 128, 2>(p, st); \
        if (p.epi == EPI_SWIGLU) return launch_t<2, BNv, EPI_SWIGLU, 128, 2>(p, st); \
        if (p.epi == EPI_QKV) return launch_t<2, BNv, EPI_QKV, 128, 2>(p, st);       \
    }
        SS_GEMM_CASE_MC(128)
        SS_GEMM_CASE_MC(256)
#undef SS_GEMM_CASE_MC
        return cudaErrorInvalidValue;
    }
#define SS_GEMM_CASE(CGv, BNv)                                                      \
    if (p.cg == CGv && p.bn == BNv) {                                               \
        if (p.epi == EPI_BF16) return launch_t<CGv, BNv, EPI_BF16>(p, st);          \
        if (p.epi == EPI_RESADD) return launch_t<CGv, BNv, EPI_RESADD>(p, st);      \
        if (p.epi == EPI_F32) return launch_t<CGv, BNv, EPI_F32>(p, st);            \
        if (p.epi == EPI_SWIGLU && BNv % 64 == 0) return launch_t<CGv, (BNv % 64 == 0 ? BNv : 64), EPI_SWIGLU>(p, st); \
        if (p.epi == EPI_QKV && BNv % 64 == 0) return launch_t<CGv, (BNv % 64 == 0 ? BNv : 64), EPI_QKV>(p, st); \
    }
    if (p.cg == 1 && p.ar == 32) {
#define SS_GEMM_CASE32(BNv)                                                              \
    if (p.bn == BNv) {                                                                   \
        if (p.epi == EPI_BF16) return launch_t<1, BNv, EPI_BF16, 32>(p, st);             \
        if (p.epi == EPI_RESADD) return launch_t<1, BNv, EPI_RESADD, 32>(p, st);         \
        if (p.epi == EPI_F32) return launch_t<1, BNv, EPI_F32, 32>(p, st);               \
        if (p.epi == EPI_SWIGLU) return launch_t<1, BNv, EPI_SWIGLU, 32>(p, st);         \
        if (p.epi == EPI_QKV) return launch_t<1, BNv, EPI_QKV, 32>(p, st);               \
    }
        SS_GEMM_CASE32(64)
        SS_GEMM_CASE32(128)
        SS_GEMM_CASE32(256)
#undef SS_GEMM_CASE32
        return cudaErrorInvalidValue;
    }
    SS_GEMM_CASE(1, 128)
    SS_GEMM_CASE(1, 256)
    SS_GEMM_CASE(2, 64)
    SS_GEMM_CASE(2, 96)
    SS_GEMM_CASE(2, 128)
    SS_GEMM_CASE(2, 160)
    SS_GEMM_CASE(2, 192)
    SS_GEMM_CASE(2, 224)
    SS_GEMM_CASE(2, 256)
#undef SS_GEMM_CASE
    return cudaErrorInvalidValue;
}

}  // namespace ssk

#ifdef SS_GEMM_TRACE
extern "C" __attribute__((visibility("default"))) int ss_debug_gemm_trace(unsigned long long* out, int n) {
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    if (n <= -2) {  // select the traced epilogue: -2 all, -3 - epi only that epilogue
        const int e = n == -2 ? -1 : -3 - n;
        return cudaMemcpyToSymbol(ssk::g_trace_epi, &e, sizeof(int)) == cudaSuccess ? 0 : -1;
    }
    if (n < 0) {  // clear both tables
        static unsigned long long zeros[1024 * 16] = {};
        return cudaMemcpyToSymbol(ssk::g_gemm_trace, zeros, sizeof(unsigned long long) * 8 * 1024) == cudaSuccess &&
                       cudaMemcpyToSymbol(ssk::g_gemm_trace2, zeros, sizeof(unsigned long long) * 16 * 1024) ==
                           cudaSuccess
                   ? 0
                   : -1;
    }
    if (n > 1024) {  // second table: epilogue-warp stamps of the last segment
        return cudaMemcpyFromSymbol(out, ssk::g_gemm_trace2, sizeof(unsigned long long) * 16 * 1024) == cudaSuccess
                   ? 0
                   : -1;
    }
    return cudaMemcpyFromSymbol(out, ssk::g_gemm_trace, sizeof(unsigned long long) * 8 * (n < 1024 ? n : 1024)) ==
                   cudaSuccess
               ? 0
               : -1;
}
#endif
