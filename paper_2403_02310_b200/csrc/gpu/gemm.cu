// K3: projection GEMMs over the packed token dimension on 5th-gen tensor cores.
//
//   D[M, N] = A[M, K] . B[N, K]^T      A = activations (bf16, K-major)
//                                      B = weight shard (bf16, K-major)
//
// Persistent, warp-specialised tcgen05 kernel (one CTA per SM):
//   warp 0       TMA producer: A/B tiles (SWIZZLE_128B) into a STAGES-deep ring
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer (M=128,
//                N=BN, K=16 per instruction, fp32 accumulators in TMEM)
//   warps 2..5   epilogue: tcgen05.ld -> registers -> fused epilogue -> HBM
// Accumulators are double-buffered in TMEM so tile i's epilogue overlaps tile
// i+1's MMAs. The M tail (T = 481, 2017, ...) is handled by TMA zero fill on
// load and row masking on store, so no padding to 128 is ever materialised.
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

constexpr int BM = 128;
constexpr int BK = 64;  // 128 B of bf16: one SWIZZLE_128B row
constexpr int kThreads = 192;

template <int BN>
struct GemmCfg {
    static constexpr int STAGES = BN == 256 ? 4 : 6;
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = 2 * BN;  // double-buffered fp32 accumulators
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256;
};

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                        int N, int K, void* __restrict__ out, int ldo, int num_m, int num_tiles) {
    using Cfg = GemmCfg<BN>;
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
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int num_kb = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
        }
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                const int m0 = (t % num_m) * BM, n0 = (t / num_m) * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
                    tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, kb * BK, m0, &full[s]);
                    tma_load_2d(sB + s * Cfg::B_BYTES, &tmB, kb * BK, n0, &full[s]);
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t acc_ph = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                mbar_wait(&tempty[acc], acc_ph ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(sA + s * Cfg::A_BYTES);
                    const uint32_t b_addr = smem_u32(sB + s * Cfg::B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_bf16(d_tmem, umma_desc_sw128(a_addr + 32 * k), umma_desc_sw128(b_addr + 32 * k), idesc,
                                  (kb | k) != 0);
                    umma_commit(&empty[s]);  // smem slot free once these MMAs retire
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
                if (++acc == 2) {
                    acc = 0;
                    acc_ph ^= 1;
                }
            }
        }
    } else {  // ---------------------------- epilogue warps 2..5
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int acc = 0;
        uint32_t acc_ph = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            const int m0 = (t % num_m) * BM, n0 = (t / num_m) * BN;
            const int row = m0 + q * 32 + lane;
            mbar_wait(&tfull[acc], acc_ph);
            tc_fence_after();
            const uint32_t t_row = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
            if constexpr (EPI == EPI_SWIGLU) {
#pragma unroll 1
                for (int c = 0; c < BN / 32; c += 2) {
                    uint32_t g[32], u[32];
                    tmem_ld32(t_row + uint32_t(c * 32), g);
                    tmem_ld32(t_row + uint32_t((c + 1) * 32), u);
                    tmem_wait_ld();
                    const int col = n0 + c * 32;
                    if (row < M && col < N) {
                        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out) + size_t(row) * ldo + col / 2;
                        uint32_t pk[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            pk[j] = pack_bf16(silu(__uint_as_float(g[2 * j])) * __uint_as_float(u[2 * j]),
                                              silu(__uint_as_float(g[2 * j + 1])) * __uint_as_float(u[2 * j + 1]));
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            reinterpret_cast<uint4*>(o)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
                    }
                }
            } else {
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t v[32];
                    tmem_ld32(t_row + uint32_t(c * 32), v);
                    tmem_wait_ld();
                    const int col = n0 + c * 32;
                    if (row < M && col < N) {
                        if constexpr (EPI == EPI_BF16) {
                            __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out) + size_t(row) * ldo + col;
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                reinterpret_cast<uint4*>(o)[j] = make_uint4(
                                    pack_bf16(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1])),
                                    pack_bf16(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                                    pack_bf16(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                                    pack_bf16(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
                        } else if constexpr (EPI == EPI_RESADD) {
                            float4* o = reinterpret_cast<float4*>(static_cast<float*>(out) + size_t(row) * ldo + col);
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                float4 x = o[j];
                                x.x += __uint_as_float(v[4 * j + 0]);
                                x.y += __uint_as_float(v[4 * j + 1]);
                                x.z += __uint_as_float(v[4 * j + 2]);
                                x.w += __uint_as_float(v[4 * j + 3]);
                                o[j] = x;
                            }
                        } else {  // EPI_F32
                            float4* o = reinterpret_cast<float4*>(static_cast<float*>(out) + size_t(row) * ldo + col);
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                o[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                   __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_ph ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<GemmCfg<BN>::TMEM_COLS>(tmem_base);
    }
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

template <int BN, int EPI>
cudaError_t launch_t(const GemmPlan& p, cudaStream_t st) {
    using Cfg = GemmCfg<BN>;
    static bool attr_set = false;
    auto kern = gemm_tcgen05_kernel<BN, EPI>;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int num_m = (p.M + BM - 1) / BM;
    const int num_n = (p.N + BN - 1) / BN;
    const int tiles = num_m * num_n;
    const int grid = tiles < p.num_sms ? tiles : p.num_sms;
    kern<<<grid, kThreads, Cfg::SMEM, st>>>(p.tmA, p.tmB, p.M, p.N, p.K, p.out, p.ldo, num_m, tiles);
    return cudaGetLastError();
}

}  // namespace

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

int gemm_pick_bn(int M, int N, int num_sms) {
    if (const char* f = getenv("SS_GEMM_BN")) {  // tuning override (dev only)
        const int bn = atoi(f);
        if (bn == 128 || bn == 256) return bn;
    }
    auto cost = [&](int bn) {
        const long tiles = long((M + BM - 1) / BM) * ((N + bn - 1) / bn);
        const long waves = (tiles + num_sms - 1) / num_sms;
        return double(waves) * bn * (bn == 128 ? 1.08 : 1.0);  // small per-tile overhead penalty
    };
    return cost(128) < cost(256) ? 128 : 256;
}

bool gemm_prepare(GemmPlan& p, const void* A, uint64_t a_rows, const void* B, int M, int N, int K, void* out,
                  int ldo, int epi, int num_sms, int bn) {
    if (M < 1 || N < 32 || K < 16 || N % 32 || K % 8 || (epi == EPI_SWIGLU && N % 64)) return false;
    p.M = M;
    p.N = N;
    p.K = K;
    p.out = out;
    p.ldo = ldo;
    p.epi = epi;
    p.num_sms = num_sms;
    p.bn = bn ? bn : gemm_pick_bn(M, N, num_sms);
    if (!make_tmap_2d(&p.tmA, A, a_rows, uint64_t(K), BM, BK)) return false;
    if (!make_tmap_2d(&p.tmB, B, uint64_t(N), uint64_t(K), uint32_t(p.bn), BK)) return false;
    return true;
}

cudaError_t gemm_launch(const GemmPlan& p, cudaStream_t st) {
#define SS_GEMM_CASE(BNv, E) \
    if (p.bn == BNv && p.epi == E) return launch_t<BNv, E>(p, st);
    SS_GEMM_CASE(128, EPI_BF16)
    SS_GEMM_CASE(128, EPI_RESADD)
    SS_GEMM_CASE(128, EPI_SWIGLU)
    SS_GEMM_CASE(128, EPI_F32)
    SS_GEMM_CASE(256, EPI_BF16)
    SS_GEMM_CASE(256, EPI_RESADD)
    SS_GEMM_CASE(256, EPI_SWIGLU)
    SS_GEMM_CASE(256, EPI_F32)
#undef SS_GEMM_CASE
    return cudaErrorInvalidValue;
}

}  // namespace ssk
