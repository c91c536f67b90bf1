// TMA delivery microbenchmark (dev tool, not part of the library): how many
// bytes/s can TMA deliver into shared memory chip-wide, unicast vs
// .multicast::cluster, at cluster sizes 1/2/4? Decides whether sharing GEMM
// operand tiles across CTA pairs by multicast can beat the ~12.5 TB/s L2->SM
// fill rate that bounds the M=512 GEMM main loop.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_mc scripts/tma_mc_bench.cu -lcuda
//
// Each CTA streams ITERS stages of a 256 x 64 bf16 tile (32 KB) through a
// 4-stage ring; the consumer only releases stages. mode 0: every CTA loads the
// whole tile itself (CTAs of a cluster load the SAME rows: what L2 dedup can
// do); mode 1: CTA r loads 1/CS of the tile multicast to all CS CTAs; mode 2:
// unicast, every CTA distinct rows.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e = (x);                                                      \
        if (e != cudaSuccess) {                                                   \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                              \
        }                                                                         \
    } while (0)

constexpr int STAGES = 4, TILE_ROWS = 256, TILE_BYTES = TILE_ROWS * 128, K = 4096, DISTINCT = 16;

__device__ __forceinline__ uint32_t s32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t crank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(s32(b)), "r"(ph)
        : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    while (!try_wait(b, ph)) {
    }
}

__global__ void __launch_bounds__(64) stream_kernel(const __grid_constant__ CUtensorMap tm, int iters, int mode,
                                                     int cs) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* buf = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE_BYTES);
    uint64_t* empty = full + STAGES;
    const uint32_t r = crank(), c = cid();
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(&empty[s])), "r"(mode == 1 ? cs : 1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    csync();
    const int rowblk = mode == 2 ? int((c * cs + r) % (DISTINCT * 4)) : int(c % DISTINCT);
    const int part_rows = TILE_ROWS / cs;
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters; ++i) {
            const int s = i % STAGES;
            if (i >= STAGES) wait(&empty[s], ((i / STAGES) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[s])),
                         "r"(TILE_BYTES)
                         : "memory");
            const int col = (i * 64) % K;
            if (mode == 1) {
                const uint16_t mask = uint16_t((1u << cs) - 1);
                // this CTA's slice of the tile, multicast to every CTA of the cluster
                const int row0 = rowblk * TILE_ROWS + int(r) * part_rows;
                for (int q = 0; q < part_rows / 32; ++q)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::"
                        "cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(s32(buf + s * TILE_BYTES +
                                                                             (int(r) * part_rows + q * 32) * 128)),
                        "l"(&tm), "r"(col), "r"(row0 + q * 32), "r"(s32(&full[s])), "h"(mask)
                        : "memory");
            } else {
                for (int q = 0; q < TILE_ROWS / 32; ++q)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                        "%3}], [%4];" ::"r"(s32(buf + s * TILE_BYTES + q * 32 * 128)),
                        "l"(&tm), "r"(col), "r"(rowblk * TILE_ROWS + q * 32), "r"(s32(&full[s]))
                        : "memory");
            }
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < iters; ++i) {
            const int s = i % STAGES;
            wait(&full[s], (i / STAGES) & 1);
            if (mode == 1) {
                for (int d = 0; d < cs; ++d) {
                    uint32_t a;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(s32(&empty[s])), "r"(d));
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
                }
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[s])) : "memory");
            }
        }
    }
    __syncthreads();
    csync();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    const int rows = TILE_ROWS * DISTINCT * 4;
    void* mat;
    CK(cudaMalloc(&mat, size_t(rows) * K * 2));
    CK(cudaMemset(mat, 0, size_t(rows) * K * 2));
    CUtensorMap tm;
    cuuint64_t dims[2] = {K, cuuint64_t(rows)}, strides[1] = {K * 2};
    cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, mat, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
        printf("encode failed\n");
        return 1;
    }
    const int smem = STAGES * TILE_BYTES + 2 * STAGES * 8;
    CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int cs : {1, 2, 4, 8}) {
        for (int mode : {0, 1, 2}) {
            if (cs == 1 && mode == 1) continue;
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.blockDim = dim3(64);
            cfg.dynamicSmemBytes = smem;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cfg.gridDim = dim3(cs * 64);
            int ncl = 0;
            CK(cudaOccupancyMaxActiveClusters(&ncl, stream_kernel, &cfg));
            cfg.gridDim = dim3(ncl * cs);
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                CK(cudaLaunchKernelEx(&cfg, stream_kernel, tm, iters, mode, cs));
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double delivered = double(ncl) * cs * iters * TILE_BYTES;
                const double fetched = mode == 1 ? delivered / cs : delivered;
                if (rep == 2)
                    printf("cs=%d mode=%s ctas=%d: %.3f ms, delivered %.2f TB/s, issued %.2f TB/s\n", cs,
                           mode == 0 ? "uc-shared" : mode == 1 ? "multicast" : "uc-distinct", ncl * cs, ms,
                           delivered / ms / 1e9, fetched / ms / 1e9);
            }
        }
    }
    return 0;
}
