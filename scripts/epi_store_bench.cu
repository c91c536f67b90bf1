// Residual-add epilogue store pattern in isolation (dev microbenchmark): why does one 32-column
// chunk of the GEMM's RESADD epilogue take microseconds inside the kernels?
// Each warp of CTAS x 8 warps walks 4 chunks of a 32-row x 256-column tile of x (fp32,
// row stride ld) exactly as the epilogue does: 8 x float4 residual loads per lane (coalesced
// layout: lane -> row 4j + lane/8, 16-byte column group lane%8), add, store x (float4) and the
// bf16 copy xb (8 B), per-row sums of squares by 3 shuffles, one fp32 store per row and chunk.
// Reports the median per-chunk time (globaltimer) per mode: 0 full, 1 no stores, 2 no loads,
// 3 x stores only, 4 loads + stores without xb/ssq.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/epi_store_bench scripts/epi_store_bench.cu
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
    for (int mode = 0; mode < 5; ++mode) {
        std::vector<double> all;
        for (int rep = 0; rep < 5; ++rep) {
            if (mode != 4) cudaMemset(flush, rep, size_t(512) << 20);  // x cold (HBM)
            else epi_kernel<<<ctas * 2, 256>>>(x, xb, ssq, ld, 0, out);  // x warm
            epi_kernel<<<ctas * 2, 256>>>(x, xb, ssq, ld, mode == 4 ? 0 : mode, out);
            cudaDeviceSynchronize();
            cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
            for (auto v : h) all.push_back(v / 1e3);
        }
        std::sort(all.begin(), all.end());
        printf("mode %d %-36s per-chunk us: median %.2f  p90 %.2f  max %.2f\n", mode, names[mode], all[all.size() / 2],
               all[all.size() * 9 / 10], all.back());
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
