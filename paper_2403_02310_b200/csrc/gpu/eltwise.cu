// K2 (paged KV append) and K4 (RMSNorm, RoPE, residual, argmax) plus the
// synthetic initialisers. All are HBM-bound: 16-byte vector accesses along the
// contiguous hidden / head dimension, warp-shuffle reductions.
#include "../../../include/ss_synth.h"
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace ssk {

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void embed_kernel(const int32_t* __restrict__ tokens, const __nv_bfloat16* __restrict__ table,
                             float* __restrict__ x, __nv_bfloat16* __restrict__ xb, float* __restrict__ ssq, int h,
                             uint32_t* __restrict__ epoch_ctr, uint32_t epoch_stride) {
    // The forward's first kernel: the previous forward is complete (PDL completion chain)
    // before any later kernel of this one may start — the attention producers read cached
    // K/V pages before their own grid-dependency wait — and its epochs are no longer read.
    pdl_wait();
    pdl_launch_dependents();
    if (epoch_ctr && blockIdx.x == 0 && threadIdx.x == 0) *epoch_ctr += epoch_stride;
    const int t = blockIdx.x;
    const uint4* src = reinterpret_cast<const uint4*>(table + size_t(tokens[t]) * h);
    float4* dst = reinterpret_cast<float4*>(x + size_t(t) * h);
    uint4* dxb = reinterpret_cast<uint4*>(xb + size_t(t) * h);
    // 8 elements per thread; 4 consecutive threads cover one 32-column chunk
    for (int i = threadIdx.x; i < h / 8; i += blockDim.x) {
        const uint4 v = src[i];
        const float4 a = make_float4(bf16_lo(v.x), bf16_hi(v.x), bf16_lo(v.y), bf16_hi(v.y));
        const float4 b = make_float4(bf16_lo(v.z), bf16_hi(v.z), bf16_lo(v.w), bf16_hi(v.w));
        dst[2 * i] = a;
        dst[2 * i + 1] = b;
        dxb[i] = v;
        float ss = a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w + b.x * b.x + b.y * b.y + b.z * b.z + b.w * b.w;
        ss += __shfl_xor_sync(0xffffffffu, ss, 1);
        ss += __shfl_xor_sync(0xffffffffu, ss, 2);
        if ((i & 3) == 0) ssq[size_t(t) * (h / 32) + i / 4] = ss;
    }
}

// One CTA per row: out = bf16(x * rsqrt(mean(x^2) + eps) * w).
__global__ void rmsnorm_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                               __nv_bfloat16* __restrict__ out, const int32_t* __restrict__ rows, int h, float eps) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ float red[32];
    const int r = blockIdx.x;
    const int src_row = rows ? rows[r] : r;
    const float4* xr = reinterpret_cast<const float4*>(x + size_t(src_row) * h);
    float ss = 0.f;
    for (int i = threadIdx.x; i < h / 4; i += blockDim.x) {
        const float4 v = xr[i];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        v = warp_sum(v);
        if (threadIdx.x == 0) red[0] = rsqrtf(v / float(h) + eps);
    }
    __syncthreads();
    const float inv = red[0];
    const uint2* wr = reinterpret_cast<const uint2*>(w);
    uint2* o = reinterpret_cast<uint2*>(out + size_t(r) * h);
    for (int i = threadIdx.x; i < h / 4; i += blockDim.x) {
        const float4 v = xr[i];
        const uint2 ww = wr[i];
        o[i] = make_uint2(pack_bf16(v.x * inv * bf16_lo(ww.x), v.y * inv * bf16_hi(ww.x)),
                          pack_bf16(v.z * inv * bf16_lo(ww.y), v.w * inv * bf16_hi(ww.y)));
    }
}

// One CTA per token. Thread handles 2 rotation pairs (i, i + hd/2) x2 lanes of
// 4 B; q heads -> q_out, k heads -> K page, v heads copied to V page.
__global__ void rope_append_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ q_out,
                                   const int32_t* __restrict__ pos, const int64_t* __restrict__ slot,
                                   const float2* __restrict__ cs, int nq, int nkv, int hd, int bs,
                                   __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc) {
    pdl_launch_dependents();
    pdl_wait();
    const int t = blockIdx.x;
    const int half = hd / 2;
    const int p = pos[t];
    const int64_t sl = slot[t];
    const int64_t blk = sl / bs, off = sl % bs;
    const __nv_bfloat16* row = qkv + size_t(t) * (nq + 2 * nkv) * hd;
    const float2* c = cs + size_t(p) * half;
    // rotate q and k heads: pairs (i, i + half), two consecutive i per thread
    const int pairs = (nq + nkv) * (half / 2);
    for (int idx = threadIdx.x; idx < pairs; idx += blockDim.x) {
        const int hh = idx / (half / 2);
        const int i = (idx % (half / 2)) * 2;
        const __nv_bfloat16* src = row + size_t(hh) * hd;
        const uint32_t lo = *reinterpret_cast<const uint32_t*>(src + i);
        const uint32_t hi = *reinterpret_cast<const uint32_t*>(src + i + half);
        const float2 c0 = c[i], c1 = c[i + 1];  // (cos, sin)
        const float x0 = bf16_lo(lo), x1 = bf16_hi(lo), y0 = bf16_lo(hi), y1 = bf16_hi(hi);
        const uint32_t nlo = pack_bf16(x0 * c0.x - y0 * c0.y, x1 * c1.x - y1 * c1.y);
        const uint32_t nhi = pack_bf16(y0 * c0.x + x0 * c0.y, y1 * c1.x + x1 * c1.y);
        if (hh < nq) {
            __nv_bfloat16* dst = q_out + (size_t(t) * nq + hh) * hd;
            *reinterpret_cast<uint32_t*>(dst + i) = nlo;
            *reinterpret_cast<uint32_t*>(dst + i + half) = nhi;
        } else {  // the page of (block, head), row `off` stored pre-swizzled (kv_page_elem)
            __nv_bfloat16* page = kc + (size_t(blk) * nkv + (hh - nq)) * bs * hd;
            *reinterpret_cast<uint32_t*>(page + kv_page_elem(int(off), i)) = nlo;
            *reinterpret_cast<uint32_t*>(page + kv_page_elem(int(off), i + half)) = nhi;
        }
    }
    // v heads: straight copy, 16 B per thread
    const int vchunks = nkv * hd / 8;
    const __nv_bfloat16* vsrc = row + size_t(nq + nkv) * hd;
    for (int idx = threadIdx.x; idx < vchunks; idx += blockDim.x) {
        const int hh = idx / (hd / 8), c8 = (idx % (hd / 8)) * 8;
        *reinterpret_cast<uint4*>(vc + (size_t(blk) * nkv + hh) * bs * hd + kv_page_elem(int(off), c8)) =
            *reinterpret_cast<const uint4*>(vsrc + size_t(hh) * hd + c8);
    }
}

__global__ void residual_add_kernel(float* __restrict__ x, const __nv_bfloat16* __restrict__ part,
                                    __nv_bfloat16* __restrict__ xb, float* __restrict__ ssq, int64_t n8, int h) {
    pdl_launch_dependents();
    pdl_wait();
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;  // multiple of 32
    for (int64_t base = blockIdx.x * int64_t(blockDim.x); base < n8; base += stride) {
        const int64_t i = base + threadIdx.x;
        const bool act = i < n8;
        float ss = 0.f;
        if (act) {
            const uint4 v = reinterpret_cast<const uint4*>(part)[i];
            float4* d = reinterpret_cast<float4*>(x) + 2 * i;
            float4 a = d[0], b = d[1];
            a.x += bf16_lo(v.x); a.y += bf16_hi(v.x); a.z += bf16_lo(v.y); a.w += bf16_hi(v.y);
            b.x += bf16_lo(v.z); b.y += bf16_hi(v.z); b.z += bf16_lo(v.w); b.w += bf16_hi(v.w);
            d[0] = a;
            d[1] = b;
            reinterpret_cast<uint4*>(xb)[i] =
                make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
            ss = a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w + b.x * b.x + b.y * b.y + b.z * b.z + b.w * b.w;
        }
        ss += __shfl_xor_sync(0xffffffffu, ss, 1);
        ss += __shfl_xor_sync(0xffffffffu, ss, 2);
        if (act && (i & 3) == 0) {  // 4 threads = one 32-column chunk of one row
            const int64_t row = i / (h / 8), g = i % (h / 8);
            ssq[row * (h / 32) + g / 4] = ss;
        }
    }
}

// ---- CUDA-IPC tensor parallelism: one-shot all-reduce fused with the residual add.
// Every rank's row-parallel GEMM wrote its bf16 partial into its own exchange buffer;
// after a flag barrier over peer memory each rank reads all ranks' partials (NVLink
// P2P loads, fixed rank order: the sum is bitwise identical on every rank), adds them in
// fp32 to the residual and emits the bf16 copy and per-chunk sums of squares.
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// The forward's device epoch base (written by embed, read after pdl_wait).
__device__ __forceinline__ uint32_t ipc_epoch_base(const IpcPeers& pe) {
    return pe.epoch_base ? *reinterpret_cast<const volatile uint32_t*>(pe.epoch_base) : 0u;
}

// Returns false (CTA-uniform) when a peer missed the collective: the error word is set
// and the caller skips its work, so a stalled rank surfaces as a status, not a trap.
__device__ __forceinline__ bool ipc_barrier(const IpcPeers& pe, uint32_t epoch) {
    __shared__ int ok;
    // one thread per CTA: CTA 0 signals every rank (its own flag slot in each rank's
    // array), then every CTA waits for all ranks' flags of this epoch
    if (threadIdx.x == 0) {
        ok = 1;
        if (blockIdx.x == 0) {
            __threadfence_system();
            for (int r = 0; r < pe.n; ++r)
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pe.flags[r] + pe.rank), "r"(epoch) : "memory");
        }
        const uint64_t t0 = globaltimer_ns();
        for (int r = 0; r < pe.n && ok; ++r) {
            uint32_t v;
            for (int spin = 0;; ++spin) {
                asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(pe.flags[pe.rank] + r) : "memory");
                if (int32_t(v - epoch) >= 0) break;
                if ((spin & 255) == 255 && globaltimer_ns() - t0 > pe.timeout_ns) {
                    atomicCAS(pe.err, 0u, kDevErrPeerTimeout | (uint32_t(r) << 8));
                    ok = 0;
                    break;
                }
            }
        }
    }
    __syncthreads();
    return ok != 0;
}

__global__ void ipc_allreduce_residual_kernel(float* __restrict__ x, const IpcPeers pe, int slot, uint32_t epoch,
                                              __nv_bfloat16* __restrict__ xb, float* __restrict__ ssq, int64_t n8,
                                              int h) {
    pdl_launch_dependents();
    pdl_wait();  // this rank's partial is complete
    if (!ipc_barrier(pe, epoch + ipc_epoch_base(pe))) return;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;  // multiple of 32
    for (int64_t base = blockIdx.x * int64_t(blockDim.x); base < n8; base += stride) {
        const int64_t i = base + threadIdx.x;
        const bool act = i < n8;
        float ss = 0.f;
        if (act) {
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
            for (int r = 0; r < pe.n; ++r) {
                const uint4 v = __ldcv(reinterpret_cast<const uint4*>(pe.buf[r][slot]) + i);
                a.x += bf16_lo(v.x); a.y += bf16_hi(v.x); a.z += bf16_lo(v.y); a.w += bf16_hi(v.y);
                b.x += bf16_lo(v.z); b.y += bf16_hi(v.z); b.z += bf16_lo(v.w); b.w += bf16_hi(v.w);
            }
            float4* d = reinterpret_cast<float4*>(x) + 2 * i;
            float4 xa = d[0], xc = d[1];
            xa.x += a.x; xa.y += a.y; xa.z += a.z; xa.w += a.w;
            xc.x += b.x; xc.y += b.y; xc.z += b.z; xc.w += b.w;
            d[0] = xa;
            d[1] = xc;
            reinterpret_cast<uint4*>(xb)[i] =
                make_uint4(pack_bf16(xa.x, xa.y), pack_bf16(xa.z, xa.w), pack_bf16(xc.x, xc.y), pack_bf16(xc.z, xc.w));
            ss = xa.x * xa.x + xa.y * xa.y + xa.z * xa.z + xa.w * xa.w + xc.x * xc.x + xc.y * xc.y + xc.z * xc.z +
                 xc.w * xc.w;
        }
        ss += __shfl_xor_sync(0xffffffffu, ss, 1);
        ss += __shfl_xor_sync(0xffffffffu, ss, 2);
        if (act && (i & 3) == 0) {  // 4 threads = one 32-column chunk of one row
            const int64_t row = i / (h / 8), g = i % (h / 8);
            ssq[row * (h / 32) + g / 4] = ss;
        }
    }
}

// Two-shot phase 1: sum this rank's share [lo, hi) of the uint4 (8 x bf16) units over every
// rank's partial in rank order (fp32), store it bf16 into this rank's red buffer.
__device__ __forceinline__ int64_t ipc_share(int64_t n8, int n) { return (n8 + n - 1) / n; }

__global__ void ipc_reduce_scatter_kernel(const IpcPeers pe, int slot, uint32_t epoch, int64_t n8) {
    pdl_launch_dependents();
    pdl_wait();  // this rank's partial is complete
    if (!ipc_barrier(pe, epoch + ipc_epoch_base(pe))) return;
    const int64_t share = ipc_share(n8, pe.n), lo = share * pe.rank, hi = min(n8, lo + share);
    uint4* dst = reinterpret_cast<uint4*>(pe.red[pe.rank]);
    for (int64_t i = lo + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < hi; i += int64_t(gridDim.x) * blockDim.x) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        for (int r = 0; r < pe.n; ++r) {
            const uint4 v = __ldcv(reinterpret_cast<const uint4*>(pe.buf[r][slot]) + i);
            a.x += bf16_lo(v.x); a.y += bf16_hi(v.x); a.z += bf16_lo(v.y); a.w += bf16_hi(v.y);
            b.x += bf16_lo(v.z); b.y += bf16_hi(v.z); b.z += bf16_lo(v.w); b.w += bf16_hi(v.w);
        }
        dst[i] = make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
    }
}

// Push reduce-scatter, phase 1 (SS_AR_PUSH): every rank's row-parallel GEMM already stored
// the units this rank owns into this rank's exchange buffer (landing zone [src][share], see
// EpiArgs::push), so after the barrier the reduction reads local HBM only: the same
// rank-order fp32 sum and bf16 store as ipc_reduce_scatter_kernel (bitwise identical).
__global__ void ipc_push_reduce_kernel(const IpcPeers pe, int slot, uint32_t epoch, int64_t n8) {
    pdl_launch_dependents();
    pdl_wait();  // this rank's GEMM (and its pushes) complete
    if (!ipc_barrier(pe, epoch + ipc_epoch_base(pe))) return;
    const int64_t share = ipc_share(n8, pe.n), lo = share * pe.rank, hi = min(n8, lo + share);
    const uint4* land = reinterpret_cast<const uint4*>(pe.buf[pe.rank][slot]);
    uint4* dst = reinterpret_cast<uint4*>(pe.red[pe.rank]);
    for (int64_t i = lo + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < hi; i += int64_t(gridDim.x) * blockDim.x) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        for (int r = 0; r < pe.n; ++r) {
            const uint4 v = __ldcv(land + r * share + (i - lo));
            a.x += bf16_lo(v.x); a.y += bf16_hi(v.x); a.z += bf16_lo(v.y); a.w += bf16_hi(v.y);
            b.x += bf16_lo(v.z); b.y += bf16_hi(v.z); b.z += bf16_lo(v.w); b.w += bf16_hi(v.w);
        }
        dst[i] = make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
    }
}

// Two-shot phase 2: every rank's reduced share -> residual add (+ bf16 copy, sums of squares).
__global__ void ipc_gather_residual_kernel(float* __restrict__ x, const IpcPeers pe, uint32_t epoch,
                                           __nv_bfloat16* __restrict__ xb, float* __restrict__ ssq, int64_t n8,
                                           int h) {
    pdl_launch_dependents();
    pdl_wait();  // this rank's share is stored
    if (!ipc_barrier(pe, epoch + ipc_epoch_base(pe))) return;
    const int64_t share = ipc_share(n8, pe.n);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;  // multiple of 32
    for (int64_t base = blockIdx.x * int64_t(blockDim.x); base < n8; base += stride) {
        const int64_t i = base + threadIdx.x;
        const bool act = i < n8;
        float ss = 0.f;
        if (act) {
            const uint4 v = __ldcv(reinterpret_cast<const uint4*>(pe.red[i / share]) + i);
            float4* d = reinterpret_cast<float4*>(x) + 2 * i;
            float4 xa = d[0], xc = d[1];
            xa.x += bf16_lo(v.x); xa.y += bf16_hi(v.x); xa.z += bf16_lo(v.y); xa.w += bf16_hi(v.y);
            xc.x += bf16_lo(v.z); xc.y += bf16_hi(v.z); xc.z += bf16_lo(v.w); xc.w += bf16_hi(v.w);
            d[0] = xa;
            d[1] = xc;
            reinterpret_cast<uint4*>(xb)[i] =
                make_uint4(pack_bf16(xa.x, xa.y), pack_bf16(xa.z, xa.w), pack_bf16(xc.x, xc.y), pack_bf16(xc.z, xc.w));
            ss = xa.x * xa.x + xa.y * xa.y + xa.z * xa.z + xa.w * xa.w + xc.x * xc.x + xc.y * xc.y + xc.z * xc.z +
                 xc.w * xc.w;
        }
        ss += __shfl_xor_sync(0xffffffffu, ss, 1);
        ss += __shfl_xor_sync(0xffffffffu, ss, 2);
        if (act && (i & 3) == 0) {  // 4 threads = one 32-column chunk of one row
            const int64_t row = i / (h / 8), g = i % (h / 8);
            ssq[row * (h / 32) + g / 4] = ss;
        }
    }
}

// Vocab all-gather of the LM-head shards: logits[row][r * vl + c] = rank r's shard.
__global__ void ipc_gather_logits_kernel(const IpcPeers pe, uint32_t epoch, float* __restrict__ out, int rows,
                                         int vl) {
    pdl_launch_dependents();
    pdl_wait();
    if (!ipc_barrier(pe, epoch + ipc_epoch_base(pe))) return;
    const int64_t n = int64_t(pe.n) * rows * vl;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / (int64_t(rows) * vl), rem = i % (int64_t(rows) * vl), row = rem / vl, c = rem % vl;
        out[row * int64_t(pe.n) * vl + r * vl + c] = __ldcv(pe.logits[r] + rem);
    }
}

// Greedy argmax per row; ties resolve to the lowest index.
__global__ void argmax_kernel(const float* __restrict__ logits, int V, int ld, int32_t* __restrict__ out) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ float sv[32];
    __shared__ int si[32];
    const float* r = logits + size_t(blockIdx.x) * ld;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    // 8 independent loads in flight per thread per step (the scan is latency-bound)
    const int step = blockDim.x * 8;
    for (int i0 = threadIdx.x; i0 < V; i0 += step) {
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = i0 + k * blockDim.x < V ? __ldg(r + i0 + k * blockDim.x) : -INFINITY;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = i0 + k * blockDim.x;
            if (v[k] > best || (v[k] == best && i < bi)) {  // ascending i per thread: ties keep the lowest
                best = v[k];
                bi = i;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
            best = ov;
            bi = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = best;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w)
            if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
                best = sv[w];
                bi = si[w];
            }
        out[blockIdx.x] = bi;
    }
}

__global__ void gather_vocab_kernel(const float* __restrict__ in, float* __restrict__ out, int tp, int rows, int vl) {
    pdl_launch_dependents();
    pdl_wait();
    const int64_t n = int64_t(tp) * rows * vl;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = (i / vl) % rows, k = i / (int64_t(vl) * rows), c = i % vl;
        out[r * int64_t(tp) * vl + k * vl + c] = in[i];
    }
}

// One-shot all-reduce over peer buffers: out = sum_r src[r], fp32 accumulation in
// rank order, 8 bf16 per thread per step. The sources are device pointers the
// caller can dereference (ranks of a local group on one device; the same kernel
// reads NVLink peer memory when handed IPC-mapped pointers).
__global__ void peer_sum_kernel(__nv_bfloat16* __restrict__ out, const PeerBufs src, int n_src, int64_t n8) {
    pdl_launch_dependents();
    pdl_wait();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
        float acc[8] = {};
        for (int r = 0; r < n_src; ++r) {
            const uint4 v = reinterpret_cast<const uint4*>(src.p[r])[i];
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                acc[2 * j] += bf16_lo(w[j]);
                acc[2 * j + 1] += bf16_hi(w[j]);
            }
        }
        reinterpret_cast<uint4*>(out)[i] = make_uint4(pack_bf16(acc[0], acc[1]), pack_bf16(acc[2], acc[3]),
                                                      pack_bf16(acc[4], acc[5]), pack_bf16(acc[6], acc[7]));
    }
}

// Element (i, j) of this rank's shard -> (tag, global row, global col, scale).
__global__ void init_weight_kernel(__nv_bfloat16* __restrict__ w, const WeightInit wi) {
    const int64_t n = wi.rows * wi.cols;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < n;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = idx / wi.cols, j = idx % wi.cols;
        uint32_t tag = 0;
        uint64_t gr = 0, gc = uint64_t(j);
        float sc = wi.scale_a;
        switch (wi.kind) {
            case W_QKV: {
                const int64_t qr = int64_t(wi.nq_l) * wi.hd, kr = int64_t(wi.nkv_l) * wi.hd;
                int64_t i = idx / wi.cols;  // logical row (per-head chunk order restored)
                if (wi.qkv_interleave && wi.hd == 128) {
                    const int64_t off = i % 128, k = off / 32;
                    i += ((k == 1) ? 32 : (k == 2) ? -32 : 0);  // stored chunk k holds logical chunk {0,2,1,3}[k]
                }
                if (i < qr) {
                    tag = SS_TAG_LAYER(wi.layer, SS_T_Q);
                    gr = uint64_t(wi.rank * qr + i);
                } else if (i < qr + kr) {
                    tag = SS_TAG_LAYER(wi.layer, SS_T_K);
                    gr = uint64_t(wi.rank * kr + (i - qr));
                    sc = wi.scale_b;
                } else {
                    tag = SS_TAG_LAYER(wi.layer, SS_T_V);
                    gr = uint64_t(wi.rank * kr + (i - qr - kr));
                    sc = wi.scale_c;
                }
                break;
            }
            case W_O:
                tag = SS_TAG_LAYER(wi.layer, SS_T_O);
                gr = uint64_t(i);
                gc = uint64_t(int64_t(wi.rank) * wi.cols + j);
                break;
            case W_GU: {
                const int64_t b = i / 64, r = i % 64;
                const bool gate = r < 32;
                tag = SS_TAG_LAYER(wi.layer, gate ? SS_T_GATE : SS_T_UP);
                gr = uint64_t(int64_t(wi.rank) * wi.ffn_l + b * 32 + (gate ? r : r - 32));
                sc = gate ? wi.scale_a : wi.scale_b;
                break;
            }
            case W_DOWN:
                tag = SS_TAG_LAYER(wi.layer, SS_T_DOWN);
                gr = uint64_t(i);
                gc = uint64_t(int64_t(wi.rank) * wi.cols + j);
                break;
            case W_EMBED:
                tag = SS_TAG_EMBED;
                gr = uint64_t(i);
                break;
            case W_LMHEAD:
                tag = SS_TAG_LMHEAD;
                gr = uint64_t(int64_t(wi.rank) * wi.vocab_l + i);
                break;
            default: {  // W_NORM: one gain vector [1][cols]
                w[idx] = __ushort_as_bfloat16(ss_norm_gain_bf16(wi.seed, wi.layer, wi.norm, j));
                continue;
            }
        }
        w[idx] = __ushort_as_bfloat16(ss_synth_bf16(wi.seed, tag, gr, gc, sc));
    }
}

__global__ void fold_gain_kernel(__nv_bfloat16* __restrict__ w, const __nv_bfloat16* __restrict__ g, int64_t rows,
                                 int64_t cols) {
    const int64_t n = rows * cols;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < n; idx += int64_t(gridDim.x) * blockDim.x)
        w[idx] = __float2bfloat16_rn(__bfloat162float(w[idx]) * __bfloat162float(g[idx % cols]));
}

__global__ void kv_fill_kernel(__nv_bfloat16* __restrict__ kb, __nv_bfloat16* __restrict__ vb, int64_t lstride,
                               int L, const int32_t* __restrict__ bt, int n_tokens, int rid, int nkv_l, int kv_off,
                               int nkv_g, int hd, int bs, uint64_t seed, int layer0) {
    const int64_t per_layer = int64_t(n_tokens) * nkv_l * hd;
    const int64_t n = per_layer * L * 2;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < n;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int which = int(idx / (per_layer * L));
        const int64_t rem = idx % (per_layer * L);
        const int layer = int(rem / per_layer);
        const int64_t e = rem % per_layer;
        const int pos = int(e / (int64_t(nkv_l) * hd));
        const int h = int((e / hd) % nkv_l), d = int(e % hd);
        const uint16_t v = ss_synth_kv(seed, layer0 + layer, which, rid, pos, kv_off + h, d, nkv_g, hd);
        const int64_t blk = bt[pos / bs];
        const int64_t off = layer * lstride + (blk * nkv_l + h) * bs * hd + kv_page_elem(pos % bs, d);
        (which ? vb : kb)[off] = __ushort_as_bfloat16(v);
    }
}

int grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    return int(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

}  // namespace

cudaError_t embed_launch(const int32_t* tokens, const __nv_bfloat16* table, float* x, __nv_bfloat16* xb, float* ssq,
                         int T, int h, uint32_t* epoch_ctr, uint32_t epoch_stride, cudaStream_t st) {
    return T > 0 ? launch_pdl(embed_kernel, dim3(T), dim3(256), 0, st, 1, tokens, table, x, xb, ssq, h, epoch_ctr,
                              epoch_stride)
                 : cudaSuccess;
}

cudaError_t rmsnorm_launch(const float* x, const __nv_bfloat16* w, __nv_bfloat16* out, const int32_t* rows, int M,
                           int h, float eps, cudaStream_t st) {
    return M > 0 ? launch_pdl(rmsnorm_kernel, dim3(M), dim3(h >= 4096 ? 512 : 256), 0, st, 1, x, w, out, rows, h, eps)
                 : cudaSuccess;
}

cudaError_t rope_append_launch(const __nv_bfloat16* qkv, __nv_bfloat16* q_out, const int32_t* pos, const int64_t* slot,
                               const float2* cs, int T, int nq, int nkv, int hd, int bs, __nv_bfloat16* kc,
                               __nv_bfloat16* vc, cudaStream_t st) {
    return T > 0 ? launch_pdl(rope_append_kernel, dim3(T), dim3(256), 0, st, 1, qkv, q_out, pos, slot, cs, nq, nkv, hd,
                              bs, kc, vc)
                 : cudaSuccess;
}

cudaError_t residual_add_launch(float* x, const __nv_bfloat16* part, __nv_bfloat16* xb, float* ssq, int T, int h,
                                cudaStream_t st) {
    const int64_t n8 = int64_t(T) * h / 8;
    return n8 > 0 ? launch_pdl(residual_add_kernel, dim3(grid_for(n8, 256)), dim3(256), 0, st, 1, x, part, xb, ssq, n8,
                               h)
                  : cudaSuccess;
}

cudaError_t ipc_allreduce_residual_launch(float* x, const IpcPeers& pe, int slot, uint32_t epoch,
                                          __nv_bfloat16* xb, float* ssq, int T, int h, cudaStream_t st) {
    const int64_t n8 = int64_t(T) * h / 8;
    // few CTAs: each spins once on the barrier, then strides over the rows
    const int grid = int(std::min<int64_t>(grid_for(n8, 256), 4 * 148));
    return n8 > 0 ? launch_pdl(ipc_allreduce_residual_kernel, dim3(grid), dim3(256), 0, st, 1, x, pe, slot, epoch, xb,
                               ssq, n8, h)
                  : cudaSuccess;
}

cudaError_t ipc_reduce_scatter_launch(const IpcPeers& pe, int slot, uint32_t epoch, int T, int h, cudaStream_t st) {
    const int64_t n8 = int64_t(T) * h / 8;
    const int grid = int(std::min<int64_t>(grid_for((n8 + pe.n - 1) / pe.n, 256), 4 * 148));
    return n8 > 0 ? launch_pdl(ipc_reduce_scatter_kernel, dim3(grid), dim3(256), 0, st, 1, pe, slot, epoch, n8)
                  : cudaSuccess;
}

cudaError_t ipc_push_reduce_launch(const IpcPeers& pe, int slot, uint32_t epoch, int T, int h, cudaStream_t st) {
    const int64_t n8 = int64_t(T) * h / 8;
    const int grid = int(std::min<int64_t>(grid_for((n8 + pe.n - 1) / pe.n, 256), 4 * 148));
    return n8 > 0 ? launch_pdl(ipc_push_reduce_kernel, dim3(grid), dim3(256), 0, st, 1, pe, slot, epoch, n8)
                  : cudaSuccess;
}

cudaError_t ipc_gather_residual_launch(float* x, const IpcPeers& pe, uint32_t epoch, __nv_bfloat16* xb, float* ssq,
                                       int T, int h, cudaStream_t st) {
    const int64_t n8 = int64_t(T) * h / 8;
    const int grid = int(std::min<int64_t>(grid_for(n8, 256), 4 * 148));
    return n8 > 0 ? launch_pdl(ipc_gather_residual_kernel, dim3(grid), dim3(256), 0, st, 1, x, pe, epoch, xb, ssq,
                               n8, h)
                  : cudaSuccess;
}

cudaError_t ipc_gather_logits_launch(const IpcPeers& pe, uint32_t epoch, float* out, int rows, int vl,
                                     cudaStream_t st) {
    const int64_t n = int64_t(pe.n) * rows * vl;
    const int grid = int(std::min<int64_t>(grid_for(n, 256), 4 * 148));
    return n > 0 ? launch_pdl(ipc_gather_logits_kernel, dim3(grid), dim3(256), 0, st, 1, pe, epoch, out, rows, vl)
                 : cudaSuccess;
}

cudaError_t argmax_launch(const float* logits, int rows, int V, int ld, int32_t* out, cudaStream_t st) {
    return rows > 0 ? launch_pdl(argmax_kernel, dim3(rows), dim3(512), 0, st, 1, logits, V, ld, out) : cudaSuccess;
}

cudaError_t gather_vocab_launch(const float* in, float* out, int tp, int rows, int vl, cudaStream_t st) {
    const int64_t n = int64_t(tp) * rows * vl;
    return n > 0 ? launch_pdl(gather_vocab_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, 1, in, out, tp, rows, vl)
                 : cudaSuccess;
}

cudaError_t peer_sum_launch(__nv_bfloat16* out, const PeerBufs& src, int n_src, int64_t n, cudaStream_t st) {
    const int64_t n8 = n / 8;
    return n8 > 0 ? launch_pdl(peer_sum_kernel, dim3(grid_for(n8, 256)), dim3(256), 0, st, 1, out, src, n_src, n8)
                  : cudaSuccess;
}

cudaError_t init_weight_launch(__nv_bfloat16* w, const WeightInit& wi, cudaStream_t st) {
    init_weight_kernel<<<grid_for(wi.rows * wi.cols, 256), 256, 0, st>>>(w, wi);
    return cudaGetLastError();
}

cudaError_t fold_gain_launch(__nv_bfloat16* w, const __nv_bfloat16* gain, int64_t rows, int64_t cols, cudaStream_t st) {
    fold_gain_kernel<<<grid_for(rows * cols, 256), 256, 0, st>>>(w, gain, rows, cols);
    return cudaGetLastError();
}

cudaError_t kv_fill_launch(__nv_bfloat16* kb, __nv_bfloat16* vb, int64_t lstride, int L, const int32_t* bt,
                           int n_tokens, int rid, int nkv_l, int kv_off, int nkv_g, int hd, int bs, uint64_t seed,
                           int layer0, cudaStream_t st) {
    const int64_t n = int64_t(n_tokens) * nkv_l * hd * L * 2;
    if (n > 0)
        kv_fill_kernel<<<grid_for(n, 256), 256, 0, st>>>(kb, vb, lstride, L, bt, n_tokens, rid, nkv_l, kv_off, nkv_g,
                                                         hd, bs, seed, layer0);
    return cudaGetLastError();
}

namespace {
__global__ void epoch_advance_kernel(uint32_t* ctr, uint32_t stride) {
    pdl_wait();  // the previous forward's kernels have completed (their epochs are no longer read)
    *ctr += stride;
}
}  // namespace

cudaError_t epoch_advance_launch(uint32_t* epoch_ctr, uint32_t epoch_stride, cudaStream_t st) {
    return launch_pdl(epoch_advance_kernel, dim3(1), dim3(1), 0, st, 1, epoch_ctr, epoch_stride);
}

}  // namespace ssk
