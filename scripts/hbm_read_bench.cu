// HBM read bandwidth with TMA bulk copies (dev microbenchmark): the ceiling for the
// HBM-streaming decode attention, which only reads. CTAS_PER_SM CTAs per SM each stream a
// distinct contiguous slice of a 2 GiB buffer through a STAGES x CHUNK shared-memory ring
// (cp.async.bulk, mbarrier completion; the consumer just releases stages).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/hbm_read_bench scripts/hbm_read_bench.cu -lcuda -lcublas
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <unistd.h>
#include <cublas_v2.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(s32(b)), "r"(ph) : "memory");
}

template <int STAGES, int CHUNK, int OP = CHUNK, int STRIDE = 0>
__global__ void __launch_bounds__(64) read_kernel(const uint8_t* src, size_t per_cta, uint64_t pol_first) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CHUNK);
    uint64_t* empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // STRIDE > 0: CTA b reads OP-byte pieces at base_g + b%G*OP + j*STRIDE, G = STRIDE/OP CTAs
    // interleaved over one region (the paged pool [block][head][16][hd]: a head's pages 32 KB apart)
    const int G = STRIDE ? STRIDE / OP : 1;
    const uint8_t* base = src + size_t(blockIdx.x / G) * per_cta * G + size_t(blockIdx.x % G) * OP;
    const int n = int(per_cta / CHUNK);
    if (threadIdx.x == 0) {
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            if (i >= STAGES) wait(&empty[s], ((i / STAGES) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[s])), "r"(CHUNK) : "memory");
            for (int o = 0; o < CHUNK; o += OP)  // OP-byte copies (the attention kernel issues 2 KB boxes)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(s32(smem + s * CHUNK + o)),
                             "l"(STRIDE ? base + (size_t(i) * (CHUNK / OP) + o / OP) * STRIDE
                                        : base + size_t(i) * CHUNK + o),
                             "r"(OP), "r"(s32(&full[s])) : "memory");
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            wait(&full[s], (i / STAGES) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[s])) : "memory");
        }
    }
}

// 2D tensor TMA of [rows][64] bf16 boxes of 16 rows (SWIZZLE_128B) — the decode attention's
// K/V page halves — 16 boxes per 32 KB stage, contiguous rows per CTA.
template <int STAGES>
__global__ void __launch_bounds__(64) read_tmap_kernel(const __grid_constant__ CUtensorMap tm, int rows_per_cta) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int CHUNK = 32768;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CHUNK);
    uint64_t* empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int row0 = blockIdx.x * rows_per_cta;
    const int n = rows_per_cta / 256;  // 16 boxes of 16 rows per stage
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            if (lane == 0) {
                if (i >= STAGES) wait(&empty[s], ((i / STAGES) - 1) & 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[s])), "r"(CHUNK) : "memory");
            }
            __syncwarp();
            if (lane < 16)  // one box per lane, as the attention producer issues them
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                             ::"r"(s32(smem + s * CHUNK + lane * 2048)), "l"(&tm), "r"(0), "r"(row0 + i * 256 + lane * 16),
                             "r"(s32(&full[s])) : "memory");
            __syncwarp();
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            wait(&full[s], (i / STAGES) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[s])) : "memory");
        }
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 3D view of 4 KB pages ([rows][2 halves][64] bf16, row stride 256 B): dims {64 elems, rows
// (stride 256 B), 2 halves (stride 128 B)}, box {64, 16, 2} -> one op per page landing as
// [2 halves][16 rows][128 B] (the attention tile's half-major image)
template <int STAGES>
__global__ void __launch_bounds__(64) read_tmap3_kernel(const __grid_constant__ CUtensorMap tm, int rows_per_cta) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int CHUNK = 32768;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CHUNK);
    uint64_t* empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int row0 = blockIdx.x * rows_per_cta;  // rows of 256 B
    const int n = rows_per_cta / 128;            // 8 pages (16 rows x 256 B) per 32 KB stage
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            if (lane == 0) {
                if (i >= STAGES) wait(&empty[s], ((i / STAGES) - 1) & 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[s])), "r"(CHUNK) : "memory");
            }
            __syncwarp();
            if (lane < 8)
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                             ::"r"(s32(smem + s * CHUNK + lane * 4096)), "l"(&tm), "r"(0), "r"(row0 + i * 128 + lane * 16),
                             "r"(0), "r"(s32(&full[s])) : "memory");
            __syncwarp();
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            wait(&full[s], (i / STAGES) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[s])) : "memory");
        }
    }
}

void run_tmap3(uint8_t* buf, size_t total, int sms) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    const uint64_t rows = total / 256;
    CUtensorMap tm;
    cuuint64_t dims[3] = {64, rows, 2};
    cuuint64_t strides[2] = {256, 128};
    cuuint32_t box[3] = {64, 16, 2}, es[3] = {1, 1, 1};
    CUresult r = reinterpret_cast<EncodeFn>(fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("3D tensor map encode failed (%d)\n", int(r));
        return;
    }
    auto k = read_tmap3_kernel<3>;
    const int smem = 3 * 32768 + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int ctas = 2 * sms;
    const int rows_per = int((rows / ctas) / 128 * 128);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k<<<ctas, 64, smem>>>(tm, rows_per);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    printf("3D tensor TMA, one 4 KB page (16 rows x 2 halves x 64) per op, 8 per stage x 3 x 2 CTA/SM: %.2f TB/s (%s)\n",
           double(rows_per) * 256 * ctas / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

void run_tmap(uint8_t* buf, size_t total, int sms) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    const uint64_t rows = total / 128;
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
    reinterpret_cast<EncodeFn>(fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto k = read_tmap_kernel<3>;
    const int smem = 3 * 32768 + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int ctas = 2 * sms;
    const int rows_per = int((rows / ctas) / 256 * 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k<<<ctas, 64, smem>>>(tm, rows_per);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    printf("2D tensor TMA, 16x64 bf16 SWIZZLE_128B boxes, 16 per 32 KB stage x 3 stages x 2 CTA/SM: %.2f TB/s\n",
           double(rows_per) * 128 * ctas / (best * 1e-3) / 1e12);
}

template <int STAGES, int CHUNK, int OP = CHUNK, int STRIDE = 0>
void run(const uint8_t* buf, size_t total, int ctas_per_sm, int sms) {
    auto k = read_kernel<STAGES, CHUNK, OP, STRIDE>;
    const int smem = STAGES * CHUNK + 2 * STAGES * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int ctas = ctas_per_sm * sms;
    const int G = STRIDE ? STRIDE / OP : 1;
    const int ctas_r = ctas / G * G;  // whole groups of interleaved readers
    const size_t per = (total / ctas_r) / CHUNK * CHUNK;
    uint64_t pol;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // evict-first policy as the decode K/V loads use (createpolicy on the device is simplest: pass 0 = normal)
    pol = 0;
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k<<<ctas_r, 64, smem>>>(buf, per, pol);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    printf("stages %2d x chunk %6d B (ops of %5d B%s) x %d CTA/SM (%4d KB in flight per SM): %.2f TB/s\n", STAGES,
           CHUNK, OP, STRIDE ? ", 32 KB-strided pages" : "", ctas_per_sm, STAGES * CHUNK * ctas_per_sm / 1024,
           double(per) * ctas_r / (best * 1e-3) / 1e12);
}

// The decode attention producer without the attention: CTA (seq e, head h) of NSEQ x 8 streams
// its sequence's 64 pages (4096 keys) of K and V from two paged pools ([block][8 heads][16][128]
// bf16, a sequence's blocks consecutive), a 64-key tile (4 pages x 2 halves x {K, V} = 16 ops of
// 2 KB, one per lane) per 32 KB stage, 3 stages; HINT: L2 evict-first cache hint as the kernel.
__device__ unsigned long long g_clk[4];
template <int HINT>
__global__ void __launch_bounds__(64) paged_kernel(const uint8_t* kp, const uint8_t* vp, int npages) {
    extern __shared__ __align__(1024) uint8_t smem[];
    unsigned long long c0 = clock64(), t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    constexpr int STAGES = 3, CHUNK = 32768;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CHUNK);
    uint64_t* empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int e = blockIdx.x / 8, h = blockIdx.x % 8, lane = threadIdx.x & 31;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int n = npages / 4;
    if (threadIdx.x < 32) {
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            if (i >= STAGES) wait(&empty[s], ((i / STAGES) - 1) & 1);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[s])), "r"(CHUNK) : "memory");
            __syncwarp();
            if (lane < 16) {
                const int kv = lane & 1, hh = (lane >> 1) & 1, pg = lane >> 2;
                const uint8_t* src = (kv ? vp : kp) + ((size_t(e) * npages + i * 4 + pg) * 8 + h) * 4096 + hh * 2048;
                const uint32_t dst = s32(smem + s * CHUNK + kv * 16384 + hh * 8192 + pg * 2048);
                if (HINT)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                                 ::"r"(dst), "l"(src), "r"(2048), "r"(s32(&full[s])), "l"(pol) : "memory");
                else
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(dst), "l"(src), "r"(2048), "r"(s32(&full[s])) : "memory");
            }
            __syncwarp();
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            wait(&full[s], (i / STAGES) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[s])) : "memory");
        }
        if (blockIdx.x == 0) {
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            g_clk[0] = clock64() - c0;
            g_clk[1] = t1 - t0;
        }
    }
}

template <int HINT>
void run_paged(const uint8_t* buf, int nseq, int npages) {
    auto k = paged_kernel<HINT>;
    const int smem = 100 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const size_t pool = size_t(nseq) * npages * 8 * 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 7; ++rep) {
        cudaEventRecord(e0);
        k<<<nseq * 8, 64, smem>>>(buf, buf + pool, npages);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    printf("paged K+V, %d seqs x 8 heads x %d pages%s: %6.1f us, %.2f TB/s\n", nseq, npages,
           HINT ? ", evict-first hint" : "", best * 1e3, 2.0 * pool / (best * 1e-3) / 1e12);
}

// SM clock vs HBM-streaming throughput: the paged producer pattern (decodes32 volume) timed
// right after R back-to-back cuBLAS bf16 GEMMs (8192^3) that drive the board to its power cap,
// so it runs at the clock the power controller left; the clock is read inside the kernel
// (clock64 / globaltimer of CTA 0).
void run_hot(const uint8_t* buf) {
    cublasHandle_t h;
    cublasCreate(&h);
    const int n = 8192;
    __nv_bfloat16 *A, *B, *Cm;
    cudaMalloc(&A, size_t(n) * n * 2);
    cudaMalloc(&B, size_t(n) * n * 2);
    cudaMalloc(&Cm, size_t(n) * n * 2);
    cudaMemset(A, 0, size_t(n) * n * 2);
    cudaMemset(B, 0, size_t(n) * n * 2);
    const float one = 1.f, zero = 0.f;
    auto k = paged_kernel<1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const size_t pool = size_t(32) * 256 * 8 * 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int R : {0, 0, 2, 8, 32, 128, 0, 0}) {
        if (R == 0) cudaDeviceSynchronize(), usleep(300000);  // idle: clocks recover
        for (int r = 0; r < R; ++r)
            cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, CUDA_R_16BF, n, B, CUDA_R_16BF, n, &zero, Cm,
                         CUDA_R_16BF, n, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
        cudaEventRecord(e0);
        k<<<256, 64, 100 * 1024>>>(buf, buf + pool, 256);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long c[2];
        cudaMemcpyFromSymbol(c, g_clk, sizeof(c));
        printf("after %3d GEMMs: paged K+V decodes32 %6.1f us, %.2f TB/s, SM clock %4.0f MHz, %.0f B/SM-clk\n", R,
               ms * 1e3, 2.0 * pool / (ms * 1e-3) / 1e12, double(c[0]) / double(c[1]) * 1e3,
               2.0 * pool / (ms * 1e-3) / (double(c[0]) / double(c[1]) * 1e9));
    }
    cublasDestroy(h);
}

// The decode attention's shape: NCTAS CTAs (2 resident per SM by shared memory) each streaming
// an equal slice of BYTES (decodes32: 256 (sequence, kv head) pairs x 2 MB of K+V = 537 MB).
template <int STAGES, int CHUNK, int OP>
void run_n(const uint8_t* buf, size_t bytes, int nctas) {
    auto k = read_kernel<STAGES, CHUNK, OP, 0>;
    const int smem = 100 * 1024;  // as the attention CTA: two per SM
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const size_t per = (bytes / nctas) / CHUNK * CHUNK;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 7; ++rep) {
        cudaEventRecord(e0);
        k<<<nctas, 64, smem>>>(buf, per, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    printf("%4d CTAs x %7.3f MB (3 x 32 KB ring, %d B ops): %6.1f us, %.2f TB/s\n", nctas, per / 1e6, OP, best * 1e3,
           double(per) * nctas / (best * 1e-3) / 1e12);
}

int main(int argc, char** argv) {
    if (argc > 1) {  // decode-attention occupancy shapes only
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const size_t total = size_t(2) << 30;
        uint8_t* buf;
        cudaMalloc(&buf, total);
        cudaMemset(buf, 1, total);
        const size_t b32 = size_t(256) * 4096 * 128 * 2 * 2;
        for (int n : {128, 148, 192, 256, 296, 384, 512, 592}) run_n<3, 32768, 2048>(buf, b32, n);
        for (int n : {256, 296, 512, 592}) run_n<3, 32768, 2048>(buf, 2 * b32, n);
        run_paged<0>(buf, 32, 256);
        run_paged<1>(buf, 32, 256);
        run_paged<0>(buf, 32, 512);
        run_paged<1>(buf, 32, 512);
        run_paged<0>(buf, 64, 256);
        run_paged<1>(buf, 64, 256);
        run_hot(buf);
        printf("%s\n", cudaGetErrorString(cudaGetLastError()));
        return 0;
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t total = size_t(2) << 30;
    uint8_t* buf;
    cudaMalloc(&buf, total);
    cudaMemset(buf, 1, total);
    run<3, 32768>(buf, total, 2, sms);  // the decode attention kernel's ring (2 CTAs/SM x 3 x 32 KB)
    run<4, 32768>(buf, total, 2, sms);
    run<6, 32768>(buf, total, 1, sms);
    run<6, 32768>(buf, total, 2, sms);
    run<8, 16384>(buf, total, 2, sms);
    run<3, 65536>(buf, total, 1, sms);
    run<3, 32768, 2048>(buf, total, 2, sms);  // the attention ring with its 2 KB page-half boxes
    run<3, 32768, 4096>(buf, total, 2, sms);
    run<3, 32768, 1024>(buf, total, 2, sms);
    run<3, 32768, 4096, 32768>(buf, total, 2, sms);  // a head's 4 KB pages, 8 heads interleaved per block
    run<3, 32768, 2048, 32768>(buf, total, 2, sms);
    run_tmap(buf, total, sms);
    run_tmap3(buf, total, sms);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
