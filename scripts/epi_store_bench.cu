// Residual-add epilogue store pattern in isolation (dev microbenchmark): why does one 32-column
// chunk of the GEMM's RESADD epilogue take microseconds inside the kernels?
// Each warp of CTAS x 8 warps walks 4 chunks of a 32-row x 256-column tile of x (fp32,
// row stride ld) exactly as the epilogue does: 8 x float4 residual loads per lane (coalesced
// layout: lane -> row 4j + lane/8, 16-byte column group lane%8), add, store x (float4) and the
// bf16 copy xb (8 B), per-row sums of squares by 3 shuffles, one fp32 store per row and chunk.
// Reports the median per-chunk time (globaltimer) per mode: 0 full, 1 no stores, 2 no loads,
// 3 x stores only, 4 loads + stores without xb/ssq.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/epi_store_bench scripts/epi_store_bench.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void epi_kernel(float* x, __nv_bfloat16* xb, float* ssq, int ld, int mode, unsigned long long* out) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int crow = lane >> 3, cch = lane & 7;
    // tile of this CTA: 256 rows x 256 cols; warp w: rows (w & 3) * 32 + 128 * (blockIdx.x & 1), chunks half + 2i
    const int tile_n = blockIdx.x >> 1, half = warp >> 2;
    const int rbase = (warp & 3) * 32 + 128 * (blockIdx.x & 1);
    unsigned long long t[5];
    t[0] = gt();
    for (int i = 0; i < 4; ++i) {
        const int c = half + 2 * i;
        const int col = tile_n * 256 + c * 32 + cch * 4;
        float4 xin[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int r = rbase + 4 * j + crow;
            xin[j] = mode == 2 ? make_float4(1.f, 1.f, 1.f, 1.f) : __ldcg(reinterpret_cast<const float4*>(x + size_t(r) * ld + col));
        }
        float ss[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int r = rbase + 4 * j + crow;
            float4 d = xin[j];
            d.x += 1.f;
            d.y += 1.f;
            d.z += 1.f;
            d.w += 1.f;
            ss[j] = d.x * d.x + d.y * d.y + d.z * d.z + d.w * d.w;
            if (mode != 1) {
                *reinterpret_cast<float4*>(x + size_t(r) * ld + col) = d;
                if (mode == 0 || mode == 2) {
                    __nv_bfloat162 a = __floats2bfloat162_rn(d.x, d.y), b = __floats2bfloat162_rn(d.z, d.w);
                    *reinterpret_cast<uint2*>(xb + size_t(r) * ld + col) =
                        make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
                }
            }
        }
        if (mode == 0 || mode == 2) {
#pragma unroll
            for (int m = 1; m <= 4; m <<= 1)
#pragma unroll
                for (int j = 0; j < 8; ++j) ss[j] += __shfl_xor_sync(0xffffffffu, ss[j], m);
            if (cch == 0)
#pragma unroll
                for (int j = 0; j < 8; ++j) ssq[size_t(rbase + 4 * j + crow) * (ld / 32) + col / 32] = ss[j];
        } else if (mode == 1 && ss[0] == 12345.f) {
            x[0] = ss[1];
        }
        __syncwarp();
        t[i + 1] = gt();
    }
    if (lane == 0) {
        const size_t w = size_t(blockIdx.x) * 8 + warp;
        for (int i = 0; i < 4; ++i) out[w * 4 + i] = t[i + 1] - t[i];
    }
}

__device__ __forceinline__ uint32_t s32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// Mode 5: the same chunk walk, results staged in shared memory (x: the SWIZZLE_128B image of a
// 32 x 32 fp32 box, as the GEMM epilogue's staging buffer already is; xb: a plain 32 x 64 B
// box) and written by one lane with 2D TMA stores (cp.async.bulk.tensor, bulk groups); the
// staging buffers are double-buffered per warp (wait_group.read 1 before reuse).
// PREF: residual of chunk i + 1 loaded into registers while chunk i is processed.
template <int PREF>
__global__ void epi_tma_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmxb,
                               const float* x, float* ssq, int ld, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int crow = lane >> 3, cch = lane & 7;
    const int tile_n = blockIdx.x >> 1, half = warp >> 2;
    const int rbase = (warp & 3) * 32 + 128 * (blockIdx.x & 1);
    uint8_t* wbuf = smem + warp * 2 * (4096 + 2048);
    unsigned long long t[5];
    float4 xin[2][8];
    auto load = [&](int i, float4 (&dst)[8]) {
        const int col = tile_n * 256 + (half + 2 * i) * 32 + cch * 4;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            dst[j] = __ldcg(reinterpret_cast<const float4*>(x + size_t(rbase + 4 * j + crow) * ld + col));
    };
    t[0] = gt();
    load(0, xin[0]);
    for (int i = 0; i < 4; ++i) {
        const int c = half + 2 * i;
        const int col0 = tile_n * 256 + c * 32;
        if (PREF && i + 1 < 4) load(i + 1, xin[(i + 1) & 1]);
        if (!PREF && i > 0) load(i, xin[i & 1]);
        uint8_t* bx = wbuf + (i & 1) * (4096 + 2048);
        uint8_t* bxb = bx + 4096;
        if (i >= 2) {  // the TMA stores of chunk i - 2 have read this buffer
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
        }
        float ss[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int r = 4 * j + crow;
            float4 d = xin[i & 1][j];
            d.x += 1.f;
            d.y += 1.f;
            d.z += 1.f;
            d.w += 1.f;
            ss[j] = d.x * d.x + d.y * d.y + d.z * d.z + d.w * d.w;
            *reinterpret_cast<float4*>(bx + r * 128 + ((cch ^ (r & 7)) << 4)) = d;
            __nv_bfloat162 a = __floats2bfloat162_rn(d.x, d.y), b = __floats2bfloat162_rn(d.z, d.w);
            *reinterpret_cast<uint2*>(bxb + r * 64 + cch * 8) =
                make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                         ::"l"(&tmx), "r"(col0), "r"(rbase), "r"(s32(bx)) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                         ::"l"(&tmxb), "r"(col0), "r"(rbase), "r"(s32(bxb)) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
#pragma unroll
        for (int m = 1; m <= 4; m <<= 1)
#pragma unroll
            for (int j = 0; j < 8; ++j) ss[j] += __shfl_xor_sync(0xffffffffu, ss[j], m);
        if (cch == 0)
#pragma unroll
            for (int j = 0; j < 8; ++j) ssq[size_t(rbase + 4 * j + crow) * (ld / 32) + col0 / 32] = ss[j];
        __syncwarp();
        t[i + 1] = gt();
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (lane == 0) {
        const size_t w = size_t(blockIdx.x) * 8 + warp;
        for (int i = 0; i < 4; ++i) out[w * 4 + i] = t[i + 1] - t[i];
    }
}

static void make_map(CUtensorMap* m, void* base, CUtensorMapDataType dt, int esize, int rows, int cols, int box_c,
                     CUtensorMapSwizzle sw) {
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(cols) * esize};
    cuuint32_t box[2] = {cuuint32_t(box_c), 32};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(m, dt, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("tensor map: %d\n", int(r));
}

int main() {
    const int T = 512, ld = 4096, ctas = 32;  // the O projection's 32 tiles at M = 512 (256 x 256)
    float* x;
    __nv_bfloat16* xb;
    float* ssq;
    unsigned long long* out;
    cudaMalloc(&x, size_t(T) * ld * 4);
    cudaMalloc(&xb, size_t(T) * ld * 2);
    cudaMalloc(&ssq, size_t(T) * (ld / 32) * 4);
    cudaMalloc(&out, size_t(ctas) * 8 * 4 * 8);
    cudaMemset(x, 0, size_t(T) * ld * 4);
    float* flush;
    cudaMalloc(&flush, size_t(512) << 20);
    std::vector<unsigned long long> h(size_t(ctas) * 8 * 4);
    const char* names[] = {"full (load x, store x + xb + ssq)", "loads only", "stores only (no x loads)",
                           "load x + store x", "full, x resident in L2"};
    cudaEvent_t ev0, ev1;
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    for (int mode = 0; mode < 5; ++mode) {
        std::vector<double> all, kus;
        for (int rep = 0; rep < 5; ++rep) {
            if (mode != 4) cudaMemset(flush, rep, size_t(512) << 20);  // x cold (HBM)
            else epi_kernel<<<ctas * 2, 256>>>(x, xb, ssq, ld, 0, out);  // x warm
            cudaEventRecord(ev0);
            epi_kernel<<<ctas * 2, 256>>>(x, xb, ssq, ld, mode == 4 ? 0 : mode, out);
            cudaEventRecord(ev1);
            cudaDeviceSynchronize();
            float ms;
            cudaEventElapsedTime(&ms, ev0, ev1);
            kus.push_back(ms * 1e3);
            cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
            for (auto v : h) all.push_back(v / 1e3);
        }
        std::sort(all.begin(), all.end());
        std::sort(kus.begin(), kus.end());
        printf("mode %d %-36s per-chunk us: median %.2f  p90 %.2f  max %.2f | kernel %.1f us\n", mode, names[mode],
               all[all.size() / 2], all[all.size() * 9 / 10], all.back(), kus[kus.size() / 2]);
    }
    // TMA-store epilogue (modes 5/6: no / one-chunk-ahead register prefetch; x cold)
    CUtensorMap tmx, tmxb;
    make_map(&tmx, x, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, ld, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    make_map(&tmxb, xb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, T, ld, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    const int tsm = 8 * 2 * (4096 + 2048);
    cudaFuncSetAttribute(epi_tma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, tsm);
    cudaFuncSetAttribute(epi_tma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tsm);
    for (int mode = 5; mode < 9; ++mode) {
        std::vector<double> all, kus;
        for (int rep = 0; rep < 5; ++rep) {
            if (mode < 7) cudaMemset(flush, rep, size_t(512) << 20);
            else epi_kernel<<<ctas * 2, 256>>>(x, xb, ssq, ld, 0, out);  // x warm in L2
            cudaEventRecord(ev0);
            if (mode & 1) epi_tma_kernel<0><<<ctas * 2, 256, tsm>>>(tmx, tmxb, x, ssq, ld, out);
            else epi_tma_kernel<1><<<ctas * 2, 256, tsm>>>(tmx, tmxb, x, ssq, ld, out);
            cudaEventRecord(ev1);
            cudaDeviceSynchronize();
            float ms;
            cudaEventElapsedTime(&ms, ev0, ev1);
            kus.push_back(ms * 1e3);
            cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
            for (auto v : h) all.push_back(v / 1e3);
        }
        std::sort(all.begin(), all.end());
        printf("mode %d TMA stores, %-26s per-chunk us: median %.2f  p90 %.2f  max %.2f\n", mode,
               mode == 5 ? "x cold, no prefetch" : mode == 6 ? "x cold, prefetch 1 ahead" : mode == 7 ? "x in L2, no prefetch" : "x in L2, prefetch 1 ahead",
               all[all.size() / 2], all[all.size() * 9 / 10], all.back());
        std::sort(kus.begin(), kus.end());
        printf("       kernel %.1f us\n", kus[kus.size() / 2]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
