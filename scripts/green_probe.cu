// Probe: SM-partitioned concurrency with CUDA green contexts on B200.
// Two green contexts split the SMs (A: requested count, B: the rest); a kernel on each
// green stream records (smid, start, end) per CTA into memory allocated from the
// primary context. Checks: launches succeed from the runtime API, SM sets are disjoint,
// the two kernels overlap in time, cross-stream events work, a cluster launch works,
// and a CUDA graph can be captured across the primary and green streams.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/green_probe scripts/green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <set>
#include <vector>

#define CKD(x)                                                                   \
    do {                                                                         \
        CUresult r_ = (x);                                                       \
        if (r_ != CUDA_SUCCESS) {                                                \
            const char* s = nullptr;                                             \
            cuGetErrorString(r_, &s);                                            \
            printf("FAIL %s: %s\n", #x, s ? s : "?");                            \
            return 1;                                                            \
        }                                                                        \
    } while (0)
#define CKR(x)                                                                   \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            printf("FAIL %s: %s\n", #x, cudaGetErrorString(e_));                 \
            return 1;                                                            \
        }                                                                        \
    } while (0)

__global__ void spin_kernel(unsigned long long* rec, unsigned long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
    if (threadIdx.x == 0) {
        rec[blockIdx.x * 3 + 0] = smid;
        rec[blockIdx.x * 3 + 1] = t0;
        rec[blockIdx.x * 3 + 2] = t;
    }
}

static int check(const char* name, std::vector<unsigned long long>& h, int n, std::set<unsigned>& sms,
                 unsigned long long& lo, unsigned long long& hi) {
    lo = ~0ull;
    hi = 0;
    for (int i = 0; i < n; ++i) {
        sms.insert(unsigned(h[i * 3]));
        lo = std::min(lo, h[i * 3 + 1]);
        hi = std::max(hi, h[i * 3 + 2]);
    }
    printf("%s: %d CTAs on %zu SMs, window %.1f us\n", name, n, sms.size(), (hi - lo) / 1e3);
    return 0;
}

int main(int argc, char** argv) {
    const int want = argc > 1 ? atoi(argv[1]) : 96;
    CKR(cudaSetDevice(0));
    CKR(cudaFree(0));
    CUdevice dev;
    CKD(cuDeviceGet(&dev, 0));
    CUdevResource all;
    CKD(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs %u\n", all.sm.smCount);
    CUdevResource part[1], rest;
    unsigned nb = 1;
    CKD(cuDevSmResourceSplitByCount(part, &nb, &all, &rest, 0, unsigned(want)));
    printf("split: A %u SMs, B %u SMs (groups %u)\n", part[0].sm.smCount, rest.sm.smCount, nb);
    CUdevResourceDesc dA, dB;
    CKD(cuDevResourceGenerateDesc(&dA, &part[0], 1));
    CKD(cuDevResourceGenerateDesc(&dB, &rest, 1));
    CUgreenCtx gA, gB;
    CKD(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CKD(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sA, sB;
    CKD(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, 0));
    CKD(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
    cudaStream_t main_st;
    CKR(cudaStreamCreateWithFlags(&main_st, cudaStreamNonBlocking));

    const int nA = 2 * int(part[0].sm.smCount), nB = 2 * int(rest.sm.smCount);
    unsigned long long *rA, *rB;
    CKR(cudaMalloc(&rA, size_t(nA) * 3 * 8));  // primary-context memory
    CKR(cudaMalloc(&rB, size_t(nB) * 3 * 8));
    cudaEvent_t ev0, evA, evB;
    CKR(cudaEventCreate(&ev0));
    CKR(cudaEventCreate(&evA));
    CKR(cudaEventCreate(&evB));
    // fork from the primary stream into both green streams, join back
    CKR(cudaEventRecord(ev0, main_st));
    CKR(cudaStreamWaitEvent((cudaStream_t)sA, ev0, 0));
    CKR(cudaStreamWaitEvent((cudaStream_t)sB, ev0, 0));
    spin_kernel<<<nA, 128, 0, (cudaStream_t)sA>>>(rA, 200000);
    CKR(cudaGetLastError());
    spin_kernel<<<nB, 128, 0, (cudaStream_t)sB>>>(rB, 200000);
    CKR(cudaGetLastError());
    CKR(cudaEventRecord(evA, (cudaStream_t)sA));
    CKR(cudaEventRecord(evB, (cudaStream_t)sB));
    CKR(cudaStreamWaitEvent(main_st, evA, 0));
    CKR(cudaStreamWaitEvent(main_st, evB, 0));
    CKR(cudaStreamSynchronize(main_st));
    std::vector<unsigned long long> hA(size_t(nA) * 3), hB(size_t(nB) * 3);
    CKR(cudaMemcpy(hA.data(), rA, hA.size() * 8, cudaMemcpyDeviceToHost));
    CKR(cudaMemcpy(hB.data(), rB, hB.size() * 8, cudaMemcpyDeviceToHost));
    std::set<unsigned> smA, smB;
    unsigned long long a0, a1, b0, b1;
    check("A", hA, nA, smA, a0, a1);
    check("B", hB, nB, smB, b0, b1);
    int inter = 0;
    for (unsigned s : smA) inter += smB.count(s);
    printf("SMs shared by A and B: %d; overlap of windows: %.1f us\n", inter,
           (std::min(a1, b1) > std::max(a0, b0) ? (std::min(a1, b1) - std::max(a0, b0)) / 1e3 : 0.0));

    // cluster launch (2 CTAs) on a green stream
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(8);
        cfg.blockDim = dim3(128);
        cfg.stream = (cudaStream_t)sB;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CKR(cudaLaunchKernelEx(&cfg, spin_kernel, rB, 1000ull));
        CKR(cudaStreamSynchronize((cudaStream_t)sB));
        printf("cluster launch on green stream: ok\n");
    }
    // graph capture across primary + green streams
    {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CKR(cudaStreamBeginCapture(main_st, cudaStreamCaptureModeThreadLocal));
        CKR(cudaEventRecord(ev0, main_st));
        CKR(cudaStreamWaitEvent((cudaStream_t)sA, ev0, 0));
        spin_kernel<<<nA, 128, 0, (cudaStream_t)sA>>>(rA, 1000);
        CKR(cudaEventRecord(evA, (cudaStream_t)sA));
        spin_kernel<<<4, 128, 0, main_st>>>(rB, 1000);
        CKR(cudaStreamWaitEvent(main_st, evA, 0));
        cudaError_t e = cudaStreamEndCapture(main_st, &g);
        printf("graph capture across green stream: %s\n", cudaGetErrorString(e));
        if (e == cudaSuccess) {
            e = cudaGraphInstantiate(&ge, g, 0);
            printf("instantiate: %s\n", cudaGetErrorString(e));
            if (e == cudaSuccess) {
                e = cudaGraphLaunch(ge, main_st);
                if (e == cudaSuccess) e = cudaStreamSynchronize(main_st);
                printf("graph launch: %s\n", cudaGetErrorString(e));
                if (e == cudaSuccess) {
                    CKR(cudaMemcpy(hA.data(), rA, hA.size() * 8, cudaMemcpyDeviceToHost));
                    std::set<unsigned> s2;
                    unsigned long long x0, x1;
                    check("A (graph replay)", hA, nA, s2, x0, x1);
                    int bad = 0;
                    for (unsigned s : s2) bad += smA.count(s) ? 0 : 1;
                    printf("graph replay SMs outside partition A: %d\n", bad);
                }
            }
        }
    }
    printf("DONE\n");
    return 0;
}
