// The ss_gpu.h C ABI: per-rank context (weights, paged KV pool, workspaces,
// NCCL communicator) and the hybrid-batch forward that replaces the
// reference's iteration_time() model step (reference costmodel.cpp:39-56,
// called at engine.cpp:227).
//
// Per layer, on one stream (T packed tokens, this rank's head/column shard):
//   rmsnorm(x) -> xn                                   K4
//   GEMM xn . Wqkv^T -> qkv                            K3 (tcgen05)
//   RoPE(q,k) ; append k,v to paged blocks at slot[t] K2 (+K4)
//   mixed paged attention (+ split-KV combine)        K1
//   GEMM o . Wo^T, fused residual add                  K3 (+ NCCL all-reduce when tp > 1)
//   rmsnorm(x) -> xn                                   K4
//   GEMM xn . Wgu^T, fused SiLU(gate) * up             K3
//   GEMM act . Wdown^T, fused residual add             K3 (+ NCCL all-reduce when tp > 1)
// then final norm + LM head on the logit rows only, vocab all-gather, argmax.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/ss_gpu.h"
#include "../../../include/ss_synth.h"
#include "common.cuh"
#include "kernels.cuh"

#define SS_API extern "C" __attribute__((visibility("default")))

using namespace ssk;
using bf16 = __nv_bfloat16;

namespace {

thread_local std::string g_create_err;

// ---------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*get_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    const char* (*err)(ncclResult_t) = nullptr;
    bool load(std::string& why) {
        if (h) return true;
        // Prefer an NCCL already mapped into the process (torch's), else the system one.
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            why = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
            return false;
        }
        get_id = reinterpret_cast<decltype(get_id)>(dlsym(h, "ncclGetUniqueId"));
        init_rank = reinterpret_cast<decltype(init_rank)>(dlsym(h, "ncclCommInitRank"));
        all_reduce = reinterpret_cast<decltype(all_reduce)>(dlsym(h, "ncclAllReduce"));
        all_gather = reinterpret_cast<decltype(all_gather)>(dlsym(h, "ncclAllGather"));
        destroy = reinterpret_cast<decltype(destroy)>(dlsym(h, "ncclCommDestroy"));
        err = reinterpret_cast<decltype(err)>(dlsym(h, "ncclGetErrorString"));
        if (!get_id || !init_rank || !all_reduce || !all_gather || !destroy || !err) {
            why = "libnccl.so.2 lacks required symbols";
            return false;
        }
        return true;
    }
};
Nccl g_nccl;

// TMA maps of one weight matrix, one per B-tile box height (rows staged per CTA),
// encoded on first use.
struct WMaps {
    const bf16* w = nullptr;
    int64_t rows = 0, cols = 0;
    CUtensorMap m[17];
    bool ok[17] = {};
    const CUtensorMap* get(int box_rows) {
        const int i = box_rows / 16;
        if (box_rows % 16 || i < 1 || i > 16) return nullptr;
        if (!ok[i]) ok[i] = make_tmap_2d(&m[i], w, uint64_t(rows), uint64_t(cols), uint32_t(box_rows), 64);
        return ok[i] ? &m[i] : nullptr;
    }
};

struct Layer {
    bf16 *wqkv, *wo, *wgu, *wdown, *attn_norm, *mlp_norm;
    WMaps tb_qkv, tb_o, tb_gu, tb_down;
};

// Epoch space of one forward (EpiArgs::epoch_base): more than its GEMM + collective launches.
constexpr uint32_t kEpochStride = 1u << 14;

struct GraphEnt {
    cudaGraphExec_t exec = nullptr;
    int64_t launches[SS_K_NUM_CLASSES] = {};
    int64_t total = 0;
    uint64_t last_use = 0;
};

struct Prof {
    int cls;
    cudaEvent_t a, b;
};

}  // namespace

struct ss_batch {
    int E = 0, T = 0, n_out = 0, max_blocks = 0;
    size_t dev_cap = 0;
    uint8_t* dev = nullptr;  // one allocation, sub-arrays below
    int32_t *cu_q = nullptr, *ctx_len = nullptr, *pos = nullptr, *tokens = nullptr, *bt = nullptr,
            *out_rows = nullptr;
    int64_t* slot = nullptr;
    AttnItem* items = nullptr;
    AttnCombine* combs = nullptr;
    int n_items = 0, n_combs = 0, part_rows = 0, n_tc = 0;
    int tc_mode = 0;  // AttnParams::tc of this batch
};

// Tensor parallelism on ONE device, for validating the sharded forward where only
// one GPU is visible: tp contexts share a stream, the caller drives one host
// thread per rank, and each collective is a host barrier (every rank's producer
// kernel enqueued) + a peer-sum kernel / peer copies + a second barrier (every
// reader enqueued before any rank overwrites its buffer). The kernels, shard
// math and call sequence are the tp-GPU ones; only the NCCL call differs.
struct LocalGroup {
    int n = 0, live = 0;
    cudaStream_t st = nullptr;
    std::vector<ss_ctx*> ranks;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool aborted = false;
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) return false;
        const uint64_t g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        cv.wait(lk, [&] { return gen != g || aborted; });
        return gen != g;
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu);
        aborted = true;
        cv.notify_all();
    }
    void reset() {
        std::lock_guard<std::mutex> lk(mu);
        aborted = false;
        arrived = 0;
    }
};

struct ss_ctx {
    ss_model_cfg cfg{};
    int rank = 0, tp = 1, device = 0, num_sms = 148;
    // pipeline parallelism (ss_create_pp_stage): this context holds layers
    // [layer0, layer0 + L) of cfg.num_layers; the embedding on stage 0, the final norm + LM
    // head on the last stage. ev_stage marks the end of this stage's last forward.
    int stage = 0, n_stages = 1, layer0 = 0;
    cudaEvent_t ev_stage = nullptr;
    uint64_t seed = 0;
    int h = 0, L = 0, hd = 0, nq_l = 0, nkv_l = 0, G = 1, ffn_l = 0, vocab_l = 0;
    cudaStream_t st = nullptr;
    std::string err;

    uint8_t* wmem = nullptr;
    std::vector<Layer> layers;
    bf16 *embed = nullptr, *lm_head = nullptr, *final_norm = nullptr;
    WMaps tb_lm;
    float2* rope = nullptr;

    bf16 *kc = nullptr, *vc = nullptr;
    int64_t nblocks = 0, layer_stride = 0;
    int bs = 16;

    // workspaces, capacity T_cap tokens / O_cap logit rows / P_cap partial rows
    int T_cap = 0, O_cap = 0, P_cap = 0;
    float* x = nullptr;
    bf16 *xn = nullptr, *qkv = nullptr, *q = nullptr, *o = nullptr, *act = nullptr, *part = nullptr, *xo = nullptr;
    float *logits_l = nullptr, *logits_g = nullptr, *logits = nullptr;
    int32_t* next_tok = nullptr;
    float *part_o = nullptr, *part_ml = nullptr;
    int32_t* comb_count = nullptr;  // split-KV group counters (self-resetting)
    int fused_combine = 0;          // in-kernel split merge (measured slower at 8 splits; off)
    int attn_tc = 1;                // prefill row tiles on tcgen05 (128 rows); 0: mma.sync (64 rows)
    int kv_pf_mb = 0;               // L2 warm-up of the decode K/V by idle QKV GEMM CTAs, MB (measured
                                    // neutral on the canonical batch: attention -3%, QKV +18%; off)
    int decode_split = 0;           // dev override (SS_ATTN_SPLIT): fixed keys per decode split; 0 = adaptive
    int fuse_rope = 1;              // RoPE + KV append in the QKV GEMM epilogue (else the K2 kernel)
    float* sk_part = nullptr;       // stream-K GEMM partial accumulators
    uint32_t* sk_flags = nullptr;   // stream-K ready flags: [forward GEMMs | single ss_k_gemm calls]
    uint32_t sk_epoch = 0;          // GEMM launches so far in this forward (flag epoch offset)
    uint32_t sk_single_epoch = 0;   // ss_k_gemm launches (immediate epochs, second flag half)
    // Device epoch base of the forward (EpiArgs::epoch_base, IpcPeers::epoch_base): embed adds
    // kEpochStride once per forward, every GEMM / collective launch adds its offset within the
    // forward. Graph replays therefore use fresh epochs like eager forwards do.
    uint32_t* d_epoch = nullptr;
    // CUDA graphs of the forward, one per batch shape (graph_key): captured the second time
    // a shape is seen, replayed afterwards. Invalidated when a workspace is reallocated.
    int graphs = 1;             // ss_set_graphs / SS_GRAPHS
    uint64_t ws_gen = 0;        // bumped by every workspace / batch-buffer / KV pool reallocation
    uint64_t graphs_gen = 0;
    uint64_t graph_clock = 0;
    std::map<std::vector<int64_t>, struct GraphEnt> graph_cache;
    std::map<std::vector<int64_t>, int> graph_seen;
    int64_t graph_captures = 0, graph_replays = 0;
    CUtensorMap ta_xn, ta_o, ta_act, ta_xo, ta_xb;
    CUtensorMap ta32_xn, ta32_o, ta32_act, ta32_xo, ta32_xb;  // 32-row boxes (GemmPlan::ar == 32)
    bf16* xb = nullptr;   // bf16 copy of the residual stream (A of the norm-folded GEMMs)
    float* ssq = nullptr;  // per (row, 32-column chunk) sums of squares of the residual
    // fused projection chain (gemm_chain_launch; TP = 1, T > 128): per-phase tile flags /
    // counters and K-split partials, sized for T_cap
    uint32_t* chain_flags = nullptr;
    float* chain_part = nullptr;
    size_t chain_flag_cap = 0, chain_part_cap = 0;  // flag buffer: max tiles per phase (stride)
    unsigned long long* chain_trace = nullptr;  // SS_CHAIN_TRACE: [L][kChainTraceItems][8] timeline

    uint8_t* pinned = nullptr;
    size_t pinned_cap = 0;
    ss_batch scratch;  // batch buffers reused by ss_forward_hybrid
    const ss_batch* last = nullptr;

    ncclComm_t comm = nullptr;
    LocalGroup* grp = nullptr;  // set instead of comm for a one-device TP group
    bf16* part_red = nullptr;   // local-group all-reduce result
    // CUDA-IPC transport (ss_ipc_export / ss_ipc_open): this rank's exchange region and the
    // mapped views of every rank's
    uint8_t* ipc_region = nullptr;
    size_t ipc_bytes = 0;
    int ipc_tcap = 0;
    int ipc = 0;                 // 1 once every peer is mapped
    IpcPeers ipc_peers{};
    void* ipc_mapped[kIpcMaxRanks] = {};
    uint32_t ipc_epoch = 0;      // collectives so far (identical sequence on every rank)
    uint32_t* dev_err = nullptr;   // device error word (IpcPeers::err), checked after each forward
    uint32_t* host_err = nullptr;  // pinned copy of it
    uint32_t ipc_ar = 0;         // all-reduces so far (exchange buffer = ipc_ar & 1)
    int ipc_algo = SS_AR_AUTO;   // ss_set_tp_allreduce / SS_TP_ALLREDUCE

    Tuning tu;  // dev overrides, read once at ss_create (tuning_from_env)
    // host-side microseconds of the last ss_forward_hybrid: validate + work list + staging,
    // enqueue (H2D + graph launch / eager launches + D2H), wait for the stream (ss_debug_host_times)
    double host_us[3] = {};
    bool prof = false;
    std::vector<Prof> pend;
    std::vector<cudaEvent_t> free_ev;
    double ms[SS_K_NUM_CLASSES] = {};
    int64_t launches[SS_K_NUM_CLASSES] = {};
    int64_t total_launches = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace {

ss_status fail(ss_ctx* c, ss_status s, const std::string& msg) {
    if (c) c->err = msg;
    else g_create_err = msg;
    return s;
}

// Makes ctx's device current for the duration of a C-ABI call (the caller's thread may
// have another current device) and restores the caller's.
struct DevGuard {
    int prev = -1;
    explicit DevGuard(int d) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
        else prev = -1;
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

#define CK(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? SS_OUT_OF_MEMORY : SS_CUDA_ERROR,    \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                        \
    } while (0)

#define NK(call)                                                                                    \
    do {                                                                                            \
        ncclResult_t r_ = (call);                                                                   \
        if (r_ != ncclSuccess) return fail(ctx, SS_NCCL_ERROR, std::string(#call) + ": " + g_nccl.err(r_)); \
    } while (0)

cudaEvent_t get_ev(ss_ctx* c) {
    if (!c->free_ev.empty()) {
        cudaEvent_t e = c->free_ev.back();
        c->free_ev.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Runs one launch (or a short fixed group) with optional per-class timing.
template <class F>
ss_status launch(ss_ctx* ctx, int cls, int nkernels, F&& f) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (ctx->prof) {
        a = get_ev(ctx);
        b = get_ev(ctx);
        cudaEventRecord(a, ctx->st);
    }
    cudaError_t e = f();
    if (e != cudaSuccess)
        return fail(ctx, SS_CUDA_ERROR, std::string("kernel launch (") + ss_kernel_class_name(cls) +
                                            "): " + cudaGetErrorString(e));
    if (ctx->prof) {
        cudaEventRecord(b, ctx->st);
        ctx->pend.push_back(Prof{cls, a, b});
    }
    ctx->launches[cls] += nkernels;
    ctx->total_launches += nkernels;
    return SS_OK;
}

template <class T>
T* carve(uint8_t*& p, size_t n) {
    T* r = reinterpret_cast<T*>(p);
    p += (n * sizeof(T) + 255) & ~size_t(255);
    return r;
}

ss_status init_weight(ss_ctx* ctx, bf16* w, int kind, int layer, int64_t rows, int64_t cols, float sa, float sb,
                      float sc, int norm = 0) {
    WeightInit wi{};
    wi.norm = norm;
    wi.kind = kind;
    wi.layer = layer;
    wi.rank = ctx->rank;
    wi.rows = rows;
    wi.cols = cols;
    wi.nq_l = ctx->nq_l;
    wi.nkv_l = ctx->nkv_l;
    wi.hd = ctx->hd;
    wi.qkv_interleave = ctx->fuse_rope;  // the fused QKV epilogue reads rotate-half pairs as adjacent chunks
    wi.ffn_l = ctx->ffn_l;
    wi.vocab_l = ctx->vocab_l;
    wi.seed = ctx->seed;
    wi.scale_a = sa;
    wi.scale_b = sb;
    wi.scale_c = sc;
    return init_weight_launch(w, wi, ctx->st) == cudaSuccess ? SS_OK : fail(ctx, SS_CUDA_ERROR, "weight init launch");
}

bool bmaps(WMaps& m, const bf16* w, int64_t rows, int64_t cols) {
    m.w = w;
    m.rows = rows;
    m.cols = cols;
    return m.get(128) != nullptr;  // validates the encode path once up front
}

// The fused projection chain of a layer (TP = 1, more than one 128-row tile of tokens):
// O, gate/up, down, and the next layer's QKV as one persistent launch (gemm.cu).
bool chain_enabled(const ss_ctx* ctx, int T) {
    // Tuning::chain bits: 1 CTA-pair chain (T > 128), 2 single-CTA weight-streaming chain (T <= 128)
    const int bit = T > 128 ? 1 : 2;
    return (ctx->tu.chain & bit) && ctx->tp == 1 && !ctx->grp && ctx->h % 256 == 0 && ctx->fuse_rope;
}
struct ChainDims {
    int n = 4, num_mt = 0, cg = 2, ar = 128;
    int N[4], K[4], S[4];
};
// Tiles: CTA pairs (256 rows) above 128 tokens, else single CTAs (128 rows; 32-row A stages
// up to 32 tokens). K splits: CTA pairs take about 64 k-blocks (a K = 4096 tile) per split,
// so the phases' tiles are comparable work units (down at K = 14336: 4 splits); single CTAs
// (weight streaming) split each phase over about one item per SM, at least 8 k-blocks each.
// SS_CHAIN_S overrides.
ChainDims chain_dims(const ss_ctx* ctx, int T) {
    ChainDims d;
    d.cg = T > 128 ? 2 : 1;
    d.ar = d.cg == 1 && T <= 32 ? 32 : 128;
    d.num_mt = (T + 128 * d.cg - 1) / (128 * d.cg);
    const int qd = ctx->nq_l * ctx->hd, qkvN = (ctx->nq_l + 2 * ctx->nkv_l) * ctx->hd;
    const int N[4] = {ctx->h, 2 * ctx->ffn_l, ctx->h, qkvN}, K[4] = {qd, ctx->h, ctx->ffn_l, ctx->h};
    for (int p = 0; p < 4; ++p) {
        d.N[p] = N[p];
        d.K[p] = K[p];
        const int nkb = (K[p] + 63) / 64;
        const int tiles = d.num_mt * ((N[p] + 255) / 256);
        const int auto_s = d.cg == 2 ? std::max(1, (nkb + 32) / 64)
                                     : std::max(1, std::min(nkb / 8, (ctx->num_sms + tiles - 1) / tiles));
        d.S[p] = ctx->tu.chain_splits[p] > 0 ? ctx->tu.chain_splits[p] : auto_s;
    }
    return d;
}
// Largest tile count of any phase. The flag buffer is laid out with this fixed stride —
// ready flags [4][maxt] | warp counters [4][maxt] | split counters [4][maxt][16] — so a slot is
// always the same kind (epoch flag or self-resetting counter) whatever the batch shape.
size_t chain_max_tiles(const ChainDims& d) {
    size_t t = 0;
    for (int p = 0; p < d.n; ++p) t = std::max(t, size_t(d.num_mt) * ((d.N[p] + 255) / 256));
    return t;
}
size_t chain_part_floats(const ChainDims& d) {
    size_t f = 0;
    for (int p = 0; p < d.n; ++p)
        if (d.S[p] > 1) f += size_t(d.num_mt) * ((d.N[p] + 255) / 256) * d.S[p] * 65536;
    return f;
}

ss_status ensure_workspace(ss_ctx* ctx, int T, int n_out, int part_rows) {
    if (T > ctx->T_cap) {
        const int cap = std::max(T, std::max(2 * ctx->T_cap, 64));
        cudaFree(ctx->x);
        cudaFree(ctx->xn);
        cudaFree(ctx->qkv);
        cudaFree(ctx->q);
        cudaFree(ctx->o);
        cudaFree(ctx->act);
        cudaFree(ctx->part);
        cudaFree(ctx->xb);
        cudaFree(ctx->ssq);
        cudaFree(ctx->part_red);
        ctx->part_red = nullptr;
        const size_t h = size_t(ctx->h), qd = size_t(ctx->nq_l) * ctx->hd;
        const size_t qkvd = size_t(ctx->nq_l + 2 * ctx->nkv_l) * ctx->hd;
        CK(cudaMalloc(&ctx->x, size_t(cap) * h * 4));
        CK(cudaMalloc(&ctx->xn, size_t(cap) * h * 2));
        CK(cudaMalloc(&ctx->qkv, size_t(cap) * qkvd * 2));
        CK(cudaMalloc(&ctx->q, size_t(cap) * qd * 2));
        CK(cudaMalloc(&ctx->o, size_t(cap) * qd * 2));
        CK(cudaMalloc(&ctx->act, size_t(cap) * ctx->ffn_l * 2));
        CK(cudaMalloc(&ctx->part, size_t(cap) * h * 2));
        CK(cudaMalloc(&ctx->xb, size_t(cap) * h * 2));
        CK(cudaMalloc(&ctx->ssq, size_t(cap) * (h / 32) * 4));
        if (ctx->grp) CK(cudaMalloc(&ctx->part_red, size_t(cap) * h * 2));
        ctx->T_cap = cap;
        ++ctx->ws_gen;
        if (!make_tmap_2d(&ctx->ta_xn, ctx->xn, cap, h, 128, 64) ||
            !make_tmap_2d(&ctx->ta_o, ctx->o, cap, qd, 128, 64) ||
            !make_tmap_2d(&ctx->ta_act, ctx->act, cap, ctx->ffn_l, 128, 64) ||
            !make_tmap_2d(&ctx->ta_xb, ctx->xb, cap, h, 128, 64) ||
            !make_tmap_2d(&ctx->ta32_xn, ctx->xn, cap, h, 32, 64) ||
            !make_tmap_2d(&ctx->ta32_o, ctx->o, cap, qd, 32, 64) ||
            !make_tmap_2d(&ctx->ta32_act, ctx->act, cap, ctx->ffn_l, 32, 64) ||
            !make_tmap_2d(&ctx->ta32_xb, ctx->xb, cap, h, 32, 64))
            return fail(ctx, SS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (activation maps)");
    }
    if (n_out > ctx->O_cap) {
        const int cap = std::max(n_out, std::max(2 * ctx->O_cap, 64));
        cudaFree(ctx->xo);
        cudaFree(ctx->logits_l);
        cudaFree(ctx->logits_g);
        cudaFree(ctx->logits);
        cudaFree(ctx->next_tok);
        CK(cudaMalloc(&ctx->xo, size_t(cap) * ctx->h * 2));
        CK(cudaMalloc(&ctx->logits_l, size_t(cap) * ctx->vocab_l * 4));
        if (ctx->tp > 1) {
            CK(cudaMalloc(&ctx->logits_g, size_t(cap) * ctx->vocab_l * ctx->tp * 4));
            CK(cudaMalloc(&ctx->logits, size_t(cap) * ctx->cfg.vocab * 4));
        }
        CK(cudaMalloc(&ctx->next_tok, size_t(cap) * 4));
        ctx->O_cap = cap;
        ++ctx->ws_gen;
        if (!make_tmap_2d(&ctx->ta_xo, ctx->xo, cap, ctx->h, 128, 64) ||
            !make_tmap_2d(&ctx->ta32_xo, ctx->xo, cap, ctx->h, 32, 64))
            return fail(ctx, SS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (logit rows)");
    }
    if (part_rows > ctx->P_cap) {
        const int cap = std::max(part_rows, 2 * ctx->P_cap);
        cudaFree(ctx->part_o);
        cudaFree(ctx->part_ml);
        cudaFree(ctx->comb_count);
        CK(cudaMalloc(&ctx->part_o, size_t(cap) * ctx->hd * 4));
        CK(cudaMalloc(&ctx->part_ml, size_t(cap) * 2 * 4));
        CK(cudaMalloc(&ctx->comb_count, size_t(cap) * 4));
        CK(cudaMemsetAsync(ctx->comb_count, 0, size_t(cap) * 4, ctx->st));
        ctx->P_cap = cap;
        ++ctx->ws_gen;
    }
    if (chain_enabled(ctx, T)) {  // flags must start zeroed (counters self-reset)
        const ChainDims d = chain_dims(ctx, T), dc = chain_dims(ctx, ctx->T_cap);
        const size_t maxt = std::max(chain_max_tiles(d), chain_max_tiles(dc));
        const size_t pf = std::max(chain_part_floats(d), chain_part_floats(dc));
        if (maxt > ctx->chain_flag_cap) {
            cudaFree(ctx->chain_flags);
            ctx->chain_flags = nullptr;
            CK(cudaMalloc(&ctx->chain_flags, maxt * 4 * 18 * 4));
            CK(cudaMemsetAsync(ctx->chain_flags, 0, maxt * 4 * 18 * 4, ctx->st));
            ctx->chain_flag_cap = maxt;
            ++ctx->ws_gen;
        }
        if (pf > ctx->chain_part_cap) {
            cudaFree(ctx->chain_part);
            ctx->chain_part = nullptr;
            CK(cudaMalloc(&ctx->chain_part, pf * 4));
            ctx->chain_part_cap = pf;
            ++ctx->ws_gen;
        }
    }
    return SS_OK;
}

// Work list of the mixed attention launch (see attention.cu).
void build_items(const ss_ctx* ctx, const ss_batch_desc* d, std::vector<AttnItem>& items,
                 std::vector<AttnCombine>& combs, int& part_rows, int& n_tc, int& tc_mode) {
    const int G = ctx->G;
    // Tensor-core prefill flavour: with at least an SM's worth of HBM-streaming decode
    // items, compact 128-row tiles that run beside them (2); else deep 256-row tiles
    // (two 128-row halves per CTA sharing K/V, 1); 0: mma.sync 64-row tiles.
    // work estimates in 64-key tile iterations: decode (HBM streaming) vs tensor-core tiles
    int dec_pairs = 0, pairs256 = 0;
    long dec_iters = 0, tc_iters = 0;
    for (int e = 0; e < d->num_entries; ++e) {
        const int ntok = d->cu_q[e + 1] - d->cu_q[e], rows = ntok * G, prefix = d->ctx_len[e] - ntok;
        if (rows <= 16) {
            dec_pairs += ctx->nkv_l;
            dec_iters += long(ctx->nkv_l) * ((d->ctx_len[e] + 63) / 64);
        } else {
            pairs256 += (rows + 255) / 256 * ctx->nkv_l;
            for (int r0 = 0; r0 < rows; r0 += 128)
                tc_iters += long(ctx->nkv_l) * ((prefix + std::min(rows, r0 + 128) / G + 63) / 64);
        }
    }
    // compact prefill tiles beside the decode kernel when the decodes fill the SMs and the
    // prefill work is small next to them (measured: chunk 480 @ 0 with 32 x 4k decodes);
    // else a deep flavour first: paired 256-row items when they alone fill the SMs, else
    // 128-row ones (chunk 480 @ 2048: deep 11.27 vs compact 11.85 ms/step; tau = 2048: paired
    // 26.37 vs compact 26.93)
    tc_mode = !ctx->attn_tc                                          ? 0
              : (dec_pairs >= ctx->num_sms && 4 * tc_iters < dec_iters) ? 2
              : pairs256 >= ctx->num_sms                             ? 1
                                                                     : 3;
    const int force = ctx->tu.attn_tc_mode;  // dev
    if (ctx->attn_tc && force >= 1 && force <= 3) tc_mode = force;
    if (tc_mode == 2 && dec_pairs == 0) tc_mode = 3;  // the compact flavour runs beside decode CTAs only
    struct Tile {
        int e, row0, nr, extent;
    };
    std::vector<Tile> tiles;
    int prefill_items = 0, decode_pairs = 0;
    for (int e = 0; e < d->num_entries; ++e) {
        const int ntok = d->cu_q[e + 1] - d->cu_q[e];
        const int prefix = d->ctx_len[e] - ntok;
        const int rows = ntok * G;
        const int tile = rows <= 16 ? 16 : (tc_mode == 1 ? 256 : tc_mode != 0 ? 128 : 64);
        for (int row0 = 0; row0 < rows; row0 += tile) {
            const int nr = std::min(tile, rows - row0);
            tiles.push_back(Tile{e, row0, nr, prefix + (row0 + nr - 1) / G + 1});
            if (nr > 16) prefill_items += ctx->nkv_l;
            else decode_pairs += ctx->nkv_l;
        }
    }
    const int long_split = prefill_items < ctx->num_sms ? 2048 : (1 << 30);
    part_rows = 0;
    for (const Tile& t : tiles) {
        // Decodes: split a (sequence, kv head) pair's keys only when there are
        // fewer pairs than SMs (one streaming CTA per SM already saturates HBM;
        // measured on the canonical batch, 256 unsplit pairs beat 768 splits +
        // combine by 2%); never below 512 keys per split.
        // SS_ATTN_SPLIT (dev) forces a fixed split length instead.
        int ns;
        if (t.nr <= 16) {
            if (ctx->decode_split > 0) {
                ns = std::max(1, (t.extent + ctx->decode_split / 2) / ctx->decode_split);
            } else {
                const int target = ctx->num_sms;
                ns = decode_pairs >= target ? 1 : (target + decode_pairs - 1) / decode_pairs;
                ns = std::max(1, std::min(ns, t.extent / 512));
            }
        } else {
            ns = long_split >= (1 << 30) ? 1 : std::max(1, (t.extent + long_split / 2) / long_split);
        }
        // balanced splits on 64-key boundaries (no 1-key tail splits)
        auto bound = [&](int s) { return s >= ns ? t.extent : int((int64_t(s) * t.extent / ns) & ~int64_t(63)); };
        for (int h = 0; h < ctx->nkv_l; ++h) {
            if (ns <= 1) {
                items.push_back(AttnItem{t.e, h, t.row0, t.nr, 0, t.extent, -1, -1});
                continue;
            }
            const int base = part_rows;
            const int ci = int(combs.size());
            for (int s = 0; s < ns; ++s)
                items.push_back(AttnItem{t.e, h, t.row0, t.nr, bound(s), bound(s + 1), base + s * t.nr, ci});
            combs.push_back(AttnCombine{t.e, h, t.row0, t.nr, ns, base, t.nr, 0});
            part_rows += ns * t.nr;
        }
    }
    // longest items first so the tail of the launch is short (SS_ATTN_ORDER=1,
    // dev: prefill row tiles first)
    const int order = ctx->tu.attn_order;
    const bool tc_items = tc_mode != 0;
    std::stable_sort(items.begin(), items.end(), [tc_items, order](const AttnItem& a, const AttnItem& b) {
        if (order == 1 && (a.nrows > 16) != (b.nrows > 16)) return a.nrows > 16;
        // per-key cost: decode streaming ~16, mma.sync row tile ~64, tcgen05 row tile ~8
        auto wt = [tc_items](const AttnItem& x) { return x.nrows <= 16 ? 16 : (tc_items ? 8 : 64); };
        const long ca = long(a.key1 - a.key0) * wt(a);
        const long cb = long(b.key1 - b.key0) * wt(b);
        return ca > cb;
    });
    // tensor-core row tiles first: they are the first of the two attention launches
    n_tc = 0;
    if (tc_items) {
        auto mid = std::stable_partition(items.begin(), items.end(), [](const AttnItem& x) { return x.nrows > 16; });
        n_tc = int(mid - items.begin());
    }
}

ss_status validate(ss_ctx* ctx, const ss_batch_desc* d) {
    if (!d || d->num_entries < 1 || d->num_tokens < 1 || !d->cu_q || !d->ctx_len || !d->pos || !d->token_ids ||
        !d->slot || !d->block_table || d->max_blocks < 1 || d->n_out < 0 || (d->n_out > 0 && !d->out_rows))
        return fail(ctx, SS_INVALID_ARG, "malformed batch descriptor");
    if (d->cu_q[0] != 0 || d->cu_q[d->num_entries] != d->num_tokens)
        return fail(ctx, SS_INVALID_ARG, "cu_q must start at 0 and end at num_tokens");
    if (ctx->nblocks == 0) return fail(ctx, SS_INVALID_ARG, "KV pool not allocated (ss_kv_alloc)");
    for (int e = 0; e < d->num_entries; ++e) {
        const int n = d->cu_q[e + 1] - d->cu_q[e];
        if (n < 1 || d->ctx_len[e] < n) return fail(ctx, SS_INVALID_ARG, "entry with no tokens or ctx < tokens");
        if (d->ctx_len[e] > int64_t(d->max_blocks) * ctx->bs || d->ctx_len[e] > ctx->cfg.max_positions)
            return fail(ctx, SS_INVALID_ARG, "context longer than block table / RoPE table");
        const int nb = (d->ctx_len[e] + ctx->bs - 1) / ctx->bs;
        for (int b = 0; b < nb; ++b) {
            const int32_t id = d->block_table[size_t(e) * d->max_blocks + b];
            if (id < 0 || id >= ctx->nblocks)
                return fail(ctx, SS_OUT_OF_KV, "block id " + std::to_string(id) + " outside the KV pool of " +
                                                   std::to_string(ctx->nblocks) + " blocks");
        }
        for (int t = d->cu_q[e]; t < d->cu_q[e + 1]; ++t) {
            const int p = d->pos[t];
            if (p != d->ctx_len[e] - n + (t - d->cu_q[e]))
                return fail(ctx, SS_INVALID_ARG, "positions must be prefix .. prefix+chunk-1 per entry");
            const int64_t want = int64_t(d->block_table[size_t(e) * d->max_blocks + p / ctx->bs]) * ctx->bs + p % ctx->bs;
            if (d->slot[t] != want) return fail(ctx, SS_INVALID_ARG, "slot disagrees with the block table");
            if (d->token_ids[t] < 0 || d->token_ids[t] >= ctx->cfg.vocab)
                return fail(ctx, SS_INVALID_ARG, "token id outside the vocabulary");
        }
    }
    for (int i = 0; i < d->n_out; ++i)
        if (d->out_rows[i] < 0 || d->out_rows[i] >= d->num_tokens) return fail(ctx, SS_INVALID_ARG, "bad out_rows");
    return SS_OK;
}

// ev_start (nullable) is recorded on the stream just before the descriptor's H2D copy, so a
// step's measured time covers copy + forward but not the host-side validation / work-list
// build / staging above it.
ss_status upload(ss_ctx* ctx, const ss_batch_desc* d, ss_batch* b, cudaEvent_t ev_start = nullptr) {
    if (ss_status s = validate(ctx, d)) return s;
    std::vector<AttnItem> items;
    std::vector<AttnCombine> combs;
    int part_rows = 0, n_tc = 0, tc_mode = 0;
    build_items(ctx, d, items, combs, part_rows, n_tc, tc_mode);
    const int E = d->num_entries, T = d->num_tokens;
    struct Seg {
        const void* src;
        size_t bytes;
    };
    const Seg segs[] = {
        {d->cu_q, size_t(E + 1) * 4},        {d->ctx_len, size_t(E) * 4},   {d->pos, size_t(T) * 4},
        {d->token_ids, size_t(T) * 4},       {d->block_table, size_t(E) * d->max_blocks * 4},
        {d->out_rows, size_t(d->n_out) * 4}, {d->slot, size_t(T) * 8},
        {items.data(), items.size() * sizeof(AttnItem)}, {combs.data(), combs.size() * sizeof(AttnCombine)},
    };
    size_t total = 0;
    for (const Seg& s : segs) total += (s.bytes + 255) & ~size_t(255);
    if (total > ctx->pinned_cap) {
        cudaFreeHost(ctx->pinned);
        ctx->pinned = nullptr;
        CK(cudaMallocHost(&ctx->pinned, total * 2));
        ctx->pinned_cap = total * 2;
    }
    if (total > b->dev_cap) {
        cudaFree(b->dev);
        b->dev = nullptr;
        CK(cudaMalloc(&b->dev, total * 2));
        b->dev_cap = total * 2;
        ++ctx->ws_gen;
    }
    // previous users of the pinned staging buffer must be done before overwrite
    CK(cudaStreamSynchronize(ctx->st));
    size_t off = 0;
    uint8_t* dptrs[9];
    for (int i = 0; i < 9; ++i) {
        if (segs[i].bytes) std::memcpy(ctx->pinned + off, segs[i].src, segs[i].bytes);
        dptrs[i] = b->dev + off;
        off += (segs[i].bytes + 255) & ~size_t(255);
    }
    if (ev_start) CK(cudaEventRecord(ev_start, ctx->st));
    CK(cudaMemcpyAsync(b->dev, ctx->pinned, total, cudaMemcpyHostToDevice, ctx->st));
    b->cu_q = reinterpret_cast<int32_t*>(dptrs[0]);
    b->ctx_len = reinterpret_cast<int32_t*>(dptrs[1]);
    b->pos = reinterpret_cast<int32_t*>(dptrs[2]);
    b->tokens = reinterpret_cast<int32_t*>(dptrs[3]);
    b->bt = reinterpret_cast<int32_t*>(dptrs[4]);
    b->out_rows = reinterpret_cast<int32_t*>(dptrs[5]);
    b->slot = reinterpret_cast<int64_t*>(dptrs[6]);
    b->items = reinterpret_cast<AttnItem*>(dptrs[7]);
    b->combs = reinterpret_cast<AttnCombine*>(dptrs[8]);
    b->E = E;
    b->T = T;
    b->n_out = d->n_out;
    b->max_blocks = d->max_blocks;
    b->n_items = int(items.size());
    b->n_tc = n_tc;
    b->tc_mode = tc_mode;
    b->n_combs = int(combs.size());
    b->part_rows = part_rows;
    return ensure_workspace(ctx, T, std::max(d->n_out, 1), part_rows);
}

AttnParams attn_params(const ss_ctx* ctx, const ss_batch* b, const bf16* q, bf16* o, int layer) {
    AttnParams p{};
    p.q = q;
    p.o = o;
    p.kc = ctx->kc + size_t(layer) * ctx->layer_stride;
    p.vc = ctx->vc + size_t(layer) * ctx->layer_stride;
    p.cu_q = b->cu_q;
    p.ctx_len = b->ctx_len;
    p.block_table = b->bt;
    p.max_blocks = b->max_blocks;
    p.items = b->items;
    p.n_items = b->n_items;
    p.n_tc = b->n_tc;
    p.wait_at_end = 0;
    p.num_sms = ctx->num_sms;
    p.kv_hint = ctx->tu.attn_l2hint;
    p.tc2_first = ctx->tu.attn_tc2_first;
    p.kv_pf_pages = ctx->tu.attn_pf_pages;
    p.part_o = ctx->part_o;
    p.part_ml = ctx->part_ml;
    p.comb_count = ctx->comb_count;
    p.fused_combine = ctx->fused_combine;
    p.tc = b->tc_mode;
    p.combines = b->combs;
    p.n_combines = b->n_combs;
    p.nq_l = ctx->nq_l;
    p.nkv_l = ctx->nkv_l;
    p.group = ctx->G;
    p.head_dim = ctx->hd;
    p.block_size = ctx->bs;
    p.layer_row0 = int64_t(layer) * ctx->nblocks * ctx->nkv_l * ctx->bs;
    p.scale_log2 = float(1.0 / std::sqrt(double(ctx->hd)) * 1.4426950408889634);
    return p;
}

ss_status gemm(ss_ctx* ctx, int cls, const CUtensorMap& ta, WMaps& tb, int M, int N, int K, void* out, int ldo,
               int epi, const EpiArgs& ea = EpiArgs()) {
    GemmPlan p;
    p.M = M;
    p.N = N;
    p.K = K;
    p.out = out;
    p.ldo = ldo;
    p.epi = epi;
    p.num_sms = ctx->num_sms;
    GemmShape s = gemm_pick(M, N, K, epi, ctx->num_sms, ctx->tu);
    {  // dev tuning: SS_GEMM_<class>=mode,bn[,splits] overrides the pick for one projection
        const int idx = cls == SS_K_GEMM_QKV ? 0 : cls == SS_K_GEMM_O ? 1 : cls == SS_K_GEMM_GATEUP ? 2
                      : cls == SS_K_GEMM_DOWN ? 3 : 4;
        const int* f = ctx->tu.gemm_force[idx];
        if (f[0] >= 0) s = GemmShape{M > 128 ? 2 : 1, f[1], f[2], f[0], M <= 32 && !ctx->tu.gemm_ar128 ? 32 : 128};
    }
    p.cg = s.cg;
    p.bn = s.bn;
    p.splits = s.splits;
    p.sk_mode = s.mode;
    p.ar = s.cg == 1 ? s.ar : 128;
    p.tmA = ta;
    if (p.ar == 32) {  // the same activation buffer through its 32-row-box map
        const CUtensorMap* twin = &ta == &ctx->ta_xn    ? &ctx->ta32_xn
                                  : &ta == &ctx->ta_o   ? &ctx->ta32_o
                                  : &ta == &ctx->ta_act ? &ctx->ta32_act
                                  : &ta == &ctx->ta_xo  ? &ctx->ta32_xo
                                  : &ta == &ctx->ta_xb  ? &ctx->ta32_xb
                                                        : nullptr;
        if (twin) p.tmA = *twin;
        else p.ar = 128;
    }
    p.mc = gemm_mc(s, M, ctx->tu);
    const CUtensorMap* mb = tb.get(p.bn / p.cg / p.mc);
    if (!mb) return fail(ctx, SS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (weight tile map)");
    p.tmB = *mb;
    p.part = ctx->sk_part;
    p.flags = ctx->sk_flags;
    p.epoch = ++ctx->sk_epoch;  // offset within the forward; + the device base (embed)
    p.force_sk = ctx->tu.gemm_sk;
    p.force_splits = ctx->tu.gemm_splits;
    p.debug = ctx->tu.gemm_debug;
    p.max_groups = ctx->tu.gemm_max_groups;
    p.dsm = ctx->tu.gemm_dsm;
    p.ea = ea;
    p.ea.l2hint = ctx->tu.gemm_l2hint;
    p.ea.epoch_base = ctx->d_epoch;
    return launch(ctx, cls, 1, [&] { return gemm_launch(p, ctx->st); });
}

// Sums this rank's partial (n bf16) over the TP group; *sum = where the result lives.
ss_status allreduce_bf16(ss_ctx* ctx, bf16* buf, size_t n, const bf16** sum) {
    if (LocalGroup* g = ctx->grp) {
        if (!g->barrier()) return fail(ctx, SS_NCCL_ERROR, "local TP group aborted by another rank");
        PeerBufs pb{};
        for (int r = 0; r < g->n; ++r) pb.p[r] = g->ranks[size_t(r)]->part;
        if (ss_status s = launch(ctx, SS_K_ALLREDUCE, 1,
                                 [&] { return peer_sum_launch(ctx->part_red, pb, g->n, int64_t(n), ctx->st); }))
            return s;
        if (!g->barrier()) return fail(ctx, SS_NCCL_ERROR, "local TP group aborted by another rank");
        *sum = ctx->part_red;
        return SS_OK;
    }
    *sum = buf;
    return launch(ctx, SS_K_ALLREDUCE, 1, [&]() -> cudaError_t {
        return g_nccl.all_reduce(buf, buf, n, ncclBfloat16, ncclSum, ctx->comm, ctx->st) == ncclSuccess
                   ? cudaSuccess
                   : cudaErrorUnknown;
    });
}

// logits_l (n_out x vocab_l, this rank's vocab shard) of every rank -> logits_g (rank-major).
ss_status allgather_logits(ss_ctx* ctx, int n_out) {
    const size_t cnt = size_t(n_out) * ctx->vocab_l;
    if (LocalGroup* g = ctx->grp) {
        if (!g->barrier()) return fail(ctx, SS_NCCL_ERROR, "local TP group aborted by another rank");
        for (int r = 0; r < g->n; ++r)
            CK(cudaMemcpyAsync(ctx->logits_g + size_t(r) * cnt, g->ranks[size_t(r)]->logits_l, cnt * 4,
                               cudaMemcpyDeviceToDevice, ctx->st));
        if (!g->barrier()) return fail(ctx, SS_NCCL_ERROR, "local TP group aborted by another rank");
        return SS_OK;
    }
    return launch(ctx, SS_K_ALLREDUCE, 1, [&]() -> cudaError_t {
        return g_nccl.all_gather(ctx->logits_l, ctx->logits_g, cnt, ncclFloat32, ctx->comm, ctx->st) == ncclSuccess
                   ? cudaSuccess
                   : cudaErrorUnknown;
    });
}

// IPC region layout: [exchange buffer 0 | exchange buffer 1 | two-shot share] (T_cap x h bf16 each) |
// logits shard (T_cap x vocab_l fp32) | flags (kIpcMaxRanks u32, 256 B slot)
// + 256 B: the push reduce-scatter's landing zone is tp x ceil(units / tp) 16-byte units
size_t ipc_buf_bytes(const ss_ctx* ctx) { return (size_t(ctx->ipc_tcap) * ctx->h * 2 + 256 + 255) & ~size_t(255); }
size_t ipc_red_off(const ss_ctx* ctx) { return 2 * ipc_buf_bytes(ctx); }
size_t ipc_logits_off(const ss_ctx* ctx) { return 3 * ipc_buf_bytes(ctx); }
size_t ipc_flags_off(const ss_ctx* ctx) {
    return ipc_logits_off(ctx) + ((size_t(ctx->ipc_tcap) * ctx->vocab_l * 4 + 255) & ~size_t(255));
}

// All-reduce algorithm of the IPC transport: one-shot (every rank pulls every partial:
// (tp - 1) messages of ingress per rank, one barrier), two-shot (reduce-scatter + all-gather:
// 2 (tp - 1) / tp messages, two barriers) or push (two-shot whose reduce-scatter traffic
// leaves from the GEMM epilogue: each output unit is stored straight into its owner rank's
// landing zone while the other tiles still run, and the reduction reads local HBM).
// Auto: push from tp = 4 and 1 MB (the same bytes and bits as two-shot), else one-shot.
int ipc_algo_for(const ss_ctx* ctx, int T) {
    if (ctx->ipc_algo != SS_AR_AUTO) return ctx->ipc_algo;
    return ctx->tp >= 4 && size_t(T) * ctx->h * 2 >= (size_t(1) << 20) ? SS_AR_PUSH : SS_AR_ONESHOT;
}

// Row-parallel projection + all-reduce + residual add over CUDA IPC: the GEMM writes this
// rank's bf16 partial into exchange buffer (all-reduce count & 1); one fused kernel then
// waits for every rank, sums all partials from peer memory in rank order and adds them.
ss_status ipc_project_allreduce(ss_ctx* ctx, int cls, const CUtensorMap& ta, WMaps& tb, int T, int K) {
    if (T > ctx->ipc_tcap) return fail(ctx, SS_INVALID_ARG, "batch larger than the IPC exchange capacity");
    const int slot = int(ctx->ipc_ar & 1u);
    bf16* mine = reinterpret_cast<bf16*>(ctx->ipc_region + slot * ipc_buf_bytes(ctx));
    const int algo = ipc_algo_for(ctx, T);
    EpiArgs ea;
    if (algo == SS_AR_PUSH) {
        ea.push_n = ctx->tp;
        ea.push_rank = ctx->rank;
        ea.push_share = (int64_t(T) * ctx->h / 8 + ctx->tp - 1) / ctx->tp;
        for (int r = 0; r < ctx->tp; ++r) ea.push[r] = const_cast<bf16*>(ctx->ipc_peers.buf[r][slot]);
    }
    if (ss_status s = gemm(ctx, cls, ta, tb, T, ctx->h, K, mine, ctx->h, EPI_BF16, ea)) return s;
    ++ctx->ipc_ar;
    if (algo == SS_AR_TWOSHOT || algo == SS_AR_PUSH) {
        const uint32_t ep1 = ++ctx->ipc_epoch, ep2 = ++ctx->ipc_epoch;
        if (ss_status s = launch(ctx, SS_K_ALLREDUCE, 1, [&] {
                return algo == SS_AR_PUSH ? ipc_push_reduce_launch(ctx->ipc_peers, slot, ep1, T, ctx->h, ctx->st)
                                          : ipc_reduce_scatter_launch(ctx->ipc_peers, slot, ep1, T, ctx->h, ctx->st);
            }))
            return s;
        return launch(ctx, SS_K_ALLREDUCE, 1, [&] {
            return ipc_gather_residual_launch(ctx->x, ctx->ipc_peers, ep2, ctx->xb, ctx->ssq, T, ctx->h, ctx->st);
        });
    }
    const uint32_t ep = ++ctx->ipc_epoch;
    return launch(ctx, SS_K_ALLREDUCE, 1, [&] {
        return ipc_allreduce_residual_launch(ctx->x, ctx->ipc_peers, slot, ep, ctx->xb, ctx->ssq, T, ctx->h, ctx->st);
    });
}

// Epilogue operands of layer l's QKV projection: the folded RMSNorm, RoPE of q/k, q to the
// attention layout, k/v appended into the paged pool at slot[t].
EpiArgs qkv_args(const ss_ctx* ctx, const ss_batch* b, int l) {
    EpiArgs ea;
    ea.ssq_in = ctx->ssq;
    ea.ssq_in_n = ctx->h / 32;
    ea.inv_dim = 1.f / float(ctx->h);
    ea.eps = ctx->cfg.rms_eps;
    ea.pos = b->pos;
    ea.slot = b->slot;
    ea.rope = ctx->rope;
    ea.q_out = ctx->q;
    ea.kc = ctx->kc + size_t(l) * ctx->layer_stride;
    ea.vc = ctx->vc + size_t(l) * ctx->layer_stride;
    ea.nq = ctx->nq_l;
    ea.nkv = ctx->nkv_l;
    ea.hd = ctx->hd;
    ea.bs = ctx->bs;
    return ea;
}

constexpr int kChainTraceItems = 4096;

// Layer l's O -> gate/up -> down projections and layer l + 1's QKV as one fused launch.
ss_status chain_launch(ss_ctx* ctx, const ss_batch* b, int l) {
    const int T = b->T, h = ctx->h;
    const ChainDims d = chain_dims(ctx, T);
    Layer& W = ctx->layers[size_t(l)];
    const int np = l + 1 < ctx->L ? 4 : 3;
    ChainPlan p;
    p.cg = d.cg;
    p.ar = d.ar;
    p.n_phases = np;
    p.M = T;
    p.num_mt = d.num_mt;
    p.num_sms = ctx->num_sms;
    p.epoch = ++ctx->sk_epoch;  // offset within the forward; + the device base (embed)
    p.epoch_base = ctx->d_epoch;
    p.debug = ctx->tu.chain_debug;
    EpiArgs norm_in;
    norm_in.ssq_in = ctx->ssq;
    norm_in.ssq_in_n = h / 32;
    norm_in.inv_dim = 1.f / float(h);
    norm_in.eps = ctx->cfg.rms_eps;
    EpiArgs res_out;
    res_out.xb_out = ctx->xb;
    res_out.ssq_out = ctx->ssq;
    struct Src {
        const CUtensorMap* a;
        WMaps* b;
        int epi, dep, res_dep, out_cols;
        void* out;
        int ldo;
        EpiArgs ea;
    };
    const bool a32 = d.ar == 32;  // the activation maps with 32-row boxes
    const Src src[4] = {
        {a32 ? &ctx->ta32_o : &ctx->ta_o, &W.tb_o, EPI_RESADD, -1, -1, 256, ctx->x, h, res_out},
        {a32 ? &ctx->ta32_xb : &ctx->ta_xb, &W.tb_gu, EPI_SWIGLU, 0, -1, 128, ctx->act, ctx->ffn_l, norm_in},
        {a32 ? &ctx->ta32_act : &ctx->ta_act, &W.tb_down, EPI_RESADD, 1, 0, 256, ctx->x, h, res_out},
        {a32 ? &ctx->ta32_xb : &ctx->ta_xb, np == 4 ? &ctx->layers[size_t(l) + 1].tb_qkv : nullptr, EPI_QKV, 2, -1,
         256, nullptr, d.N[3], np == 4 ? qkv_args(ctx, b, l + 1) : EpiArgs()},
    };
    const size_t maxt = ctx->chain_flag_cap;  // fixed stride of the flag buffer (chain_max_tiles)
    float* pt = ctx->chain_part;
    for (int i = 0; i < np; ++i) {
        ChainPhase& ph = p.ph[i];
        const CUtensorMap* mb = src[i].b->get(256 / d.cg);
        if (!mb) return fail(ctx, SS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (weight tile map)");
        p.tmA[i] = *src[i].a;
        p.tmB[i] = *mb;
        ph.N = d.N[i];
        ph.K = d.K[i];
        ph.epi = src[i].epi;
        ph.splits = d.S[i];
        ph.dep = src[i].dep;
        ph.res_dep = src[i].res_dep;
        ph.out_cols = src[i].out_cols;
        ph.out = src[i].out;
        ph.ldo = src[i].ldo;
        ph.ea = src[i].ea;
        const size_t tiles = size_t(d.num_mt) * ((d.N[i] + 255) / 256);
        if (tiles > maxt) return fail(ctx, SS_CUDA_ERROR, "chain flag buffer smaller than the batch's tiles");
        ph.ready = ctx->chain_flags + i * maxt;
        ph.rcnt = ctx->chain_flags + (4 + i) * maxt;
        ph.pcnt = ctx->chain_flags + 8 * maxt + i * maxt * 16;
        if (d.S[i] > 1) {
            ph.part = pt;
            pt += tiles * d.S[i] * 65536;
        }
    }
    gemm_chain_finalize(p);
    if (ctx->tu.chain_trace && p.total_items <= kChainTraceItems) {
        if (!ctx->chain_trace) {
            CK(cudaMalloc(&ctx->chain_trace, size_t(ctx->L) * kChainTraceItems * 16 * 8));
            CK(cudaMemset(ctx->chain_trace, 0, size_t(ctx->L) * kChainTraceItems * 16 * 8));
        }
        p.trace = ctx->chain_trace + size_t(l) * kChainTraceItems * 16;
    }
    return launch(ctx, SS_K_GEMM_CHAIN, 1, [&] { return gemm_chain_launch(p, ctx->st); });
}

ss_status enqueue_forward(ss_ctx* ctx, const ss_batch* b) {
    if (ctx->tp > 1 && !ctx->grp && !ctx->comm && !ctx->ipc)
        return fail(ctx, SS_INVALID_ARG, "tp > 1 needs an NCCL id at ss_create or the IPC transport (ss_ipc_open)");
    const int T = b->T, h = ctx->h;
    const int qkvN = (ctx->nq_l + 2 * ctx->nkv_l) * ctx->hd, qd = ctx->nq_l * ctx->hd;
    const float eps = ctx->cfg.rms_eps;
    ss_status s;
#define RUN(x)                 \
    if ((s = (x)) != SS_OK) \
        return s;
    // epoch offsets restart every forward; embed advances the device base (d_epoch)
    ctx->sk_epoch = 0;
    ctx->ipc_epoch = 0;
    if (ctx->stage == 0) {
        RUN(launch(ctx, SS_K_EMBED, 1, [&] {
            return embed_launch(b->tokens, ctx->embed, ctx->x, ctx->xb, ctx->ssq, T, h, ctx->d_epoch, kEpochStride,
                                ctx->st);
        }));
    } else {  // later pipeline stage: the residual stream came from the previous stage (ss_forward_stage_enqueue)
        RUN(launch(ctx, SS_K_EMBED, 1, [&] { return epoch_advance_launch(ctx->d_epoch, kEpochStride, ctx->st); }));
    }
    // RMSNorm is folded into the QKV / gate-up GEMMs: they consume the bf16 copy of
    // the residual (xb) and scale rows by rsqrt(mean(x^2) + eps) from the
    // per-chunk sums of squares (ssq) that embed / the residual-add epilogues
    // produce; the norm gains were folded into Wqkv / Wgu at ss_create.
    EpiArgs norm_in;
    norm_in.ssq_in = ctx->ssq;
    norm_in.ssq_in_n = h / 32;
    norm_in.inv_dim = 1.f / float(h);
    norm_in.eps = eps;
    EpiArgs res_out;
    res_out.xb_out = ctx->xb;
    res_out.ssq_out = ctx->ssq;
    const bool chain = chain_enabled(ctx, T);
    for (int l = 0; l < ctx->L; ++l) {
        Layer& W = ctx->layers[size_t(l)];
        EpiArgs qkv_ea = norm_in;  // + RoPE and the paged KV append (K2) in the epilogue
        qkv_ea.pos = b->pos;
        qkv_ea.slot = b->slot;
        qkv_ea.rope = ctx->rope;
        qkv_ea.q_out = ctx->q;
        qkv_ea.kc = ctx->kc + size_t(l) * ctx->layer_stride;
        qkv_ea.vc = ctx->vc + size_t(l) * ctx->layer_stride;
        qkv_ea.nq = ctx->nq_l;
        qkv_ea.nkv = ctx->nkv_l;
        qkv_ea.hd = ctx->hd;
        qkv_ea.bs = ctx->bs;
        // idle CTA pairs of the QKV GEMM warm L2 with the head of every decode item's K/V
        // (SS_KV_PF_MB budget; default off)
        if (ctx->kv_pf_mb > 0 && b->n_items > b->n_tc) {
            qkv_ea.pf_items = b->items + b->n_tc;
            qkv_ea.pf_n = b->n_items - b->n_tc;
            const size_t page_bytes = size_t(ctx->bs) * ctx->hd * 2;
            qkv_ea.pf_pages = int(size_t(ctx->kv_pf_mb) * 1048576 / (2 * page_bytes * size_t(qkv_ea.pf_n)));
            qkv_ea.pf_bt = b->bt;
            qkv_ea.pf_max_blocks = b->max_blocks;
            qkv_ea.pf_ctx_len = b->ctx_len;
            if (qkv_ea.pf_pages == 0) qkv_ea.pf_n = 0;
        }
        if (chain && l > 0) {
            // this layer's QKV ran in the previous layer's chain launch
        } else if (ctx->fuse_rope) {
            RUN(gemm(ctx, SS_K_GEMM_QKV, ctx->ta_xb, W.tb_qkv, T, qkvN, h, nullptr, qkvN, EPI_QKV, qkv_ea));
        } else {
            RUN(gemm(ctx, SS_K_GEMM_QKV, ctx->ta_xb, W.tb_qkv, T, qkvN, h, ctx->qkv, qkvN, EPI_BF16, norm_in));
            RUN(launch(ctx, SS_K_ROPE_APPEND, 1, [&] {
                return rope_append_launch(ctx->qkv, ctx->q, b->pos, b->slot, ctx->rope, T, ctx->nq_l, ctx->nkv_l,
                                          ctx->hd, ctx->bs, qkv_ea.kc, qkv_ea.vc, ctx->st);
            }));
        }
        const AttnParams ap = attn_params(ctx, b, ctx->q, ctx->o, l);
        // two kernels when the batch has both tensor-core prefill tiles and decode items
        const int n_attn = (ap.tc && ap.n_tc > 0 && ap.n_items > ap.n_tc) ? 2 : 1;
        RUN(launch(ctx, SS_K_ATTN, n_attn, [&] { return attention_launch(ap, ctx->st); }));
        if (b->n_combs && !ctx->fused_combine)
            RUN(launch(ctx, SS_K_ATTN_COMBINE, 1, [&] { return attention_combine_launch(ap, ctx->st); }));
        if (chain) {
            RUN(chain_launch(ctx, b, l));
            continue;
        }
        if (ctx->tp == 1) {
            RUN(gemm(ctx, SS_K_GEMM_O, ctx->ta_o, W.tb_o, T, h, qd, ctx->x, h, EPI_RESADD, res_out));
        } else if (ctx->ipc) {
            RUN(ipc_project_allreduce(ctx, SS_K_GEMM_O, ctx->ta_o, W.tb_o, T, qd));
        } else {
            RUN(gemm(ctx, SS_K_GEMM_O, ctx->ta_o, W.tb_o, T, h, qd, ctx->part, h, EPI_BF16));
            const bf16* sum = nullptr;
            RUN(allreduce_bf16(ctx, ctx->part, size_t(T) * h, &sum));
            RUN(launch(ctx, SS_K_ALLREDUCE, 1,
                       [&] { return residual_add_launch(ctx->x, sum, ctx->xb, ctx->ssq, T, h, ctx->st); }));
        }
        RUN(gemm(ctx, SS_K_GEMM_GATEUP, ctx->ta_xb, W.tb_gu, T, 2 * ctx->ffn_l, h, ctx->act, ctx->ffn_l, EPI_SWIGLU,
                 norm_in));
        if (ctx->tp == 1) {
            RUN(gemm(ctx, SS_K_GEMM_DOWN, ctx->ta_act, W.tb_down, T, h, ctx->ffn_l, ctx->x, h, EPI_RESADD, res_out));
        } else if (ctx->ipc) {
            RUN(ipc_project_allreduce(ctx, SS_K_GEMM_DOWN, ctx->ta_act, W.tb_down, T, ctx->ffn_l));
        } else {
            RUN(gemm(ctx, SS_K_GEMM_DOWN, ctx->ta_act, W.tb_down, T, h, ctx->ffn_l, ctx->part, h, EPI_BF16));
            const bf16* sum = nullptr;
            RUN(allreduce_bf16(ctx, ctx->part, size_t(T) * h, &sum));
            RUN(launch(ctx, SS_K_ALLREDUCE, 1,
                       [&] { return residual_add_launch(ctx->x, sum, ctx->xb, ctx->ssq, T, h, ctx->st); }));
        }
    }
    if (b->n_out > 0 && ctx->stage == ctx->n_stages - 1) {
        RUN(launch(ctx, SS_K_RMSNORM, 1, [&] {
            return rmsnorm_launch(ctx->x, ctx->final_norm, ctx->xo, b->out_rows, b->n_out, h, eps, ctx->st);
        }));
        float* lg = ctx->ipc ? reinterpret_cast<float*>(ctx->ipc_region + ipc_logits_off(ctx)) : ctx->logits_l;
        RUN(gemm(ctx, SS_K_LMHEAD, ctx->ta_xo, ctx->tb_lm, b->n_out, ctx->vocab_l, h, lg, ctx->vocab_l, EPI_F32));
        const float* full = ctx->logits_l;
        if (ctx->ipc) {  // every rank's vocab shard, read over peer memory after a flag barrier
            const uint32_t ep = ++ctx->ipc_epoch;
            RUN(launch(ctx, SS_K_ALLREDUCE, 1, [&] {
                return ipc_gather_logits_launch(ctx->ipc_peers, ep, ctx->logits, b->n_out, ctx->vocab_l, ctx->st);
            }));
            full = ctx->logits;
        } else if (ctx->tp > 1) {
            RUN(allgather_logits(ctx, b->n_out));
            RUN(launch(ctx, SS_K_ARGMAX, 1, [&] {
                return gather_vocab_launch(ctx->logits_g, ctx->logits, ctx->tp, b->n_out, ctx->vocab_l, ctx->st);
            }));
            full = ctx->logits;
        }
        RUN(launch(ctx, SS_K_ARGMAX, 1, [&] {
            return argmax_launch(full, b->n_out, ctx->cfg.vocab, ctx->cfg.vocab, ctx->next_tok, ctx->st);
        }));
    }
#undef RUN
    ctx->last = b;
    return SS_OK;
}

void graphs_clear(ss_ctx* ctx) {
    for (auto& kv : ctx->graph_cache) cudaGraphExecDestroy(kv.second.exec);
    ctx->graph_cache.clear();
    ctx->graph_seen.clear();
}

// Everything a captured forward bakes into its launches besides the (stable) workspace
// pointers: the batch's sizes, work-list counts and buffers, and the IPC buffer parity.
std::vector<int64_t> graph_key(const ss_ctx* ctx, const ss_batch* b) {
    return {b->T,      b->E,         b->n_out,     b->n_items,     b->n_tc, b->tc_mode, b->n_combs, b->part_rows,
            b->max_blocks, int64_t(reinterpret_cast<intptr_t>(b->dev)), int64_t(ctx->ipc_ar & 1u)};
}

// Enqueues one forward of b: a CUDA graph replay when this batch shape was captured, else
// eager launches (capturing the shape's graph the second time it is seen). Graphs are off
// for per-kernel profiling (events between launches) and for the one-device local group
// (host barriers between ranks), and on NCCL (dlopen'ed library; not captured).
ss_status run_forward(ss_ctx* ctx, const ss_batch* b) {
    if (!ctx->graphs || ctx->prof || ctx->grp || ctx->comm || ctx->n_stages > 1) return enqueue_forward(ctx, b);
    if (ctx->graphs_gen != ctx->ws_gen) {
        graphs_clear(ctx);
        ctx->graphs_gen = ctx->ws_gen;
    }
    const std::vector<int64_t> key = graph_key(ctx, b);
    ++ctx->graph_clock;
    auto it = ctx->graph_cache.find(key);
    if (it != ctx->graph_cache.end()) {
        GraphEnt& g = it->second;
        CK(cudaGraphLaunch(g.exec, ctx->st));
        g.last_use = ctx->graph_clock;
        for (int k = 0; k < SS_K_NUM_CLASSES; ++k) ctx->launches[k] += g.launches[k];
        ctx->total_launches += g.total;
        ctx->sk_epoch = 0;
        ctx->ipc_ar += uint32_t(2 * ctx->L * (ctx->ipc ? 1 : 0));  // the replayed all-reduces
        ctx->last = b;
        ++ctx->graph_replays;
        return SS_OK;
    }
    if (ctx->graph_seen.size() > 4096) ctx->graph_seen.clear();
    if (++ctx->graph_seen[key] < 2) return enqueue_forward(ctx, b);
    if (ctx->graph_cache.size() >= 64) {  // least recently used out
        auto lru = ctx->graph_cache.begin();
        for (auto i = ctx->graph_cache.begin(); i != ctx->graph_cache.end(); ++i)
            if (i->second.last_use < lru->second.last_use) lru = i;
        cudaGraphExecDestroy(lru->second.exec);
        ctx->graph_cache.erase(lru);
    }
    int64_t before[SS_K_NUM_CLASSES];
    std::memcpy(before, ctx->launches, sizeof(before));
    const int64_t total0 = ctx->total_launches;
    CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
    const ss_status s = enqueue_forward(ctx, b);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(ctx->st, &graph);
    if (s != SS_OK) {
        if (graph) cudaGraphDestroy(graph);
        return s;
    }
    if (ec != cudaSuccess) return fail(ctx, SS_CUDA_ERROR, std::string("graph capture: ") + cudaGetErrorString(ec));
    GraphEnt g;
    const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) return fail(ctx, SS_CUDA_ERROR, std::string("graph instantiate: ") + cudaGetErrorString(ei));
    for (int k = 0; k < SS_K_NUM_CLASSES; ++k) g.launches[k] = ctx->launches[k] - before[k];
    g.total = ctx->total_launches - total0;
    g.last_use = ctx->graph_clock;
    CK(cudaGraphLaunch(g.exec, ctx->st));  // the captured launches did not run
    ctx->graph_cache.emplace(key, g);
    ++ctx->graph_captures;
    return SS_OK;
}

// After a synchronize: a collective that timed out on a missing peer left a code in the
// device error word (see IpcPeers); report it once and clear it.
ss_status check_dev_err(ss_ctx* ctx) {
    if (!ctx->ipc || *ctx->host_err == 0) return SS_OK;
    const uint32_t e = *ctx->host_err;
    *ctx->host_err = 0;
    CK(cudaMemsetAsync(ctx->dev_err, 0, 4, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return fail(ctx, SS_NCCL_ERROR,
                "TP peer rank " + std::to_string(e >> 8) + " did not reach a collective within the timeout; the "
                "forward's outputs are invalid");
}

ss_status read_outputs(ss_ctx* ctx, const ss_batch* b, float* logits, int32_t* next) {
    if (ctx->stage != ctx->n_stages - 1 && (logits || next) && b->n_out > 0)
        return fail(ctx, SS_INVALID_ARG, "logits come from the last pipeline stage");
    if (b->n_out > 0) {
        const float* full = ctx->tp > 1 ? ctx->logits : ctx->logits_l;
        if (logits)
            CK(cudaMemcpyAsync(logits, full, size_t(b->n_out) * ctx->cfg.vocab * 4, cudaMemcpyDeviceToHost, ctx->st));
        if (next) CK(cudaMemcpyAsync(next, ctx->next_tok, size_t(b->n_out) * 4, cudaMemcpyDeviceToHost, ctx->st));
    }
    if (ctx->ipc) CK(cudaMemcpyAsync(ctx->host_err, ctx->dev_err, 4, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return check_dev_err(ctx);
}

void collect_prof(ss_ctx* ctx) {
    for (const Prof& p : ctx->pend) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) ctx->ms[p.cls] += ms;
        ctx->free_ev.push_back(p.a);
        ctx->free_ev.push_back(p.b);
    }
    ctx->pend.clear();
}

}  // namespace

// ============================================================================ C ABI

// Dev: the fused chain's per-item timeline of every layer (SS_CHAIN_TRACE=1 at ss_create):
// n >= 0 copies min(n, L * 4096 * 16) u64 into out; n < 0 clears it.
SS_API ss_status ss_debug_chain_trace(ss_ctx* ctx, unsigned long long* out, int64_t n) {
    if (!ctx) return SS_INVALID_ARG;
    DevGuard dg(ctx->device);
    if (!ctx->chain_trace) return fail(ctx, SS_INVALID_ARG, "no chain trace (SS_CHAIN_TRACE=1, and a chain launch)");
    const size_t total = size_t(ctx->L) * kChainTraceItems * 16;
    CK(cudaStreamSynchronize(ctx->st));
    if (n < 0) {
        CK(cudaMemset(ctx->chain_trace, 0, total * 8));
        return SS_OK;
    }
    CK(cudaMemcpy(out, ctx->chain_trace, std::min(size_t(n), total) * 8, cudaMemcpyDeviceToHost));
    return SS_OK;
}

SS_API const char* ss_kernel_class_name(int32_t k) {
    static const char* names[SS_K_NUM_CLASSES] = {"embed",   "rmsnorm", "gemm_qkv",    "rope_kv_append",
                                                  "attention", "attn_combine", "gemm_o", "gemm_gate_up",
                                                  "gemm_down", "nccl_allreduce", "lm_head", "argmax", "gemm_chain"};
    return (k >= 0 && k < SS_K_NUM_CLASSES) ? names[k] : "unknown";
}

SS_API const char* ss_last_error(ss_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

SS_API ss_status ss_nccl_unique_id(void* out) {
    ss_ctx* ctx = nullptr;
    std::string why;
    if (!g_nccl.load(why)) return fail(ctx, SS_NCCL_ERROR, why);
    ncclUniqueId id;
    NK(g_nccl.get_id(&id));
    std::memcpy(out, &id, sizeof(id));
    return SS_OK;
}

// ---------------------------------------------------------------- CUDA-IPC TP transport

SS_API ss_status ss_ipc_export(ss_ctx* ctx, int32_t max_tokens, void* handle_out) {
    if (!ctx || !handle_out || max_tokens < 1 || ctx->tp < 2 || ctx->grp)
        return fail(ctx, SS_INVALID_ARG, "ss_ipc_export needs a tp > 1 rank context and max_tokens >= 1");
    CK(cudaSetDevice(ctx->device));
    if (!ctx->ipc_region) {
        ctx->ipc_tcap = max_tokens;
        ctx->ipc_bytes = ipc_flags_off(ctx) + 256;
        CK(cudaMalloc(&ctx->ipc_region, ctx->ipc_bytes));
        CK(cudaMemset(ctx->ipc_region + ipc_flags_off(ctx), 0, 256));
    } else if (max_tokens != ctx->ipc_tcap) {
        return fail(ctx, SS_INVALID_ARG, "ss_ipc_export: capacity already set");
    }
    cudaIpcMemHandle_t hd;
    CK(cudaIpcGetMemHandle(&hd, ctx->ipc_region));
    std::memcpy(handle_out, &hd, sizeof(hd));
    return SS_OK;
}

SS_API ss_status ss_ipc_open(ss_ctx* ctx, const void* handles) {
    if (!ctx || !handles || !ctx->ipc_region) return fail(ctx, SS_INVALID_ARG, "ss_ipc_open needs ss_ipc_export first");
    if (ctx->tp > kIpcMaxRanks) return fail(ctx, SS_INVALID_ARG, "IPC transport supports up to 8 ranks");
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->st));
    IpcPeers pe{};
    pe.n = ctx->tp;
    pe.rank = ctx->rank;
    for (int r = 0; r < ctx->tp; ++r) {
        uint8_t* base = ctx->ipc_region;
        if (r != ctx->rank) {
            cudaIpcMemHandle_t hd;
            std::memcpy(&hd, static_cast<const uint8_t*>(handles) + size_t(r) * sizeof(hd), sizeof(hd));
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
            ctx->ipc_mapped[r] = p;
            base = static_cast<uint8_t*>(p);
        }
        pe.buf[r][0] = reinterpret_cast<const bf16*>(base);
        pe.buf[r][1] = reinterpret_cast<const bf16*>(base + ipc_buf_bytes(ctx));
        pe.red[r] = reinterpret_cast<bf16*>(base + ipc_red_off(ctx));
        pe.logits[r] = reinterpret_cast<const float*>(base + ipc_logits_off(ctx));
        pe.flags[r] = reinterpret_cast<uint32_t*>(base + ipc_flags_off(ctx));
    }
    if (!ctx->dev_err) {
        CK(cudaMalloc(&ctx->dev_err, 4));
        CK(cudaMallocHost(&ctx->host_err, 4));
    }
    CK(cudaMemset(ctx->dev_err, 0, 4));
    *ctx->host_err = 0;
    pe.err = ctx->dev_err;
    pe.timeout_ns = 10ull * 1000 * 1000 * 1000;  // a peer missing for 10 s is a failed rank
    pe.epoch_base = ctx->d_epoch;
    ctx->ipc_peers = pe;
    ++ctx->ws_gen;  // captured graphs predate the transport
    ctx->ipc = 1;
    return SS_OK;
}

static void group_release(LocalGroup* g) {
    if (--g->live == 0) {
        if (g->st) cudaStreamDestroy(g->st);
        delete g;
    }
}

static ss_status create_impl(const ss_model_cfg* cfg, int32_t tp_rank, int32_t tp_size, const void* nccl_id,
                             uint64_t weight_seed, int32_t device, LocalGroup* grp, ss_ctx** out, int32_t stage = 0,
                             int32_t n_stages = 1) {
    ss_ctx* ctx = nullptr;
    if (!cfg || !out) return fail(ctx, SS_INVALID_ARG, "null argument");
    const ss_model_cfg& c = *cfg;
    if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size) return fail(ctx, SS_INVALID_ARG, "bad tp rank/size");
    if (n_stages < 1 || stage < 0 || stage >= n_stages || n_stages > c.num_layers)
        return fail(ctx, SS_INVALID_ARG, "bad pipeline stage (need 0 <= stage < n_stages <= num_layers)");
    if (n_stages > 1 && tp_size > 1) return fail(ctx, SS_INVALID_ARG, "pipeline stages are tp_size 1 contexts");
    if (c.num_layers < 1 || c.hidden % 64 || c.num_q_heads % tp_size || c.num_kv_heads % tp_size ||
        c.num_q_heads % c.num_kv_heads || (c.head_dim != 64 && c.head_dim != 128) || c.ffn % (32 * tp_size) ||
        c.vocab % tp_size || (c.vocab / tp_size) % 32 || c.max_positions < 1)
        return fail(ctx, SS_INVALID_ARG,
                    "unsupported model shape (need hidden%64, heads%tp, hd in {64,128}, ffn%(32tp), vocab/tp%32)");
    if ((c.ffn / tp_size) % 64)
        return fail(ctx, SS_INVALID_ARG, "ffn shard must be a multiple of 64 (K tiling of the down projection)");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(ctx, SS_CUDA_ERROR, "no CUDA device visible: this library has no CPU fallback");
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return fail(ctx, SS_CUDA_ERROR, "bad device");
    if (prop.major != 10) return fail(ctx, SS_CUDA_ERROR, "needs an sm_100 (B200) device");

    ctx = new ss_ctx();
    ctx->cfg = c;
    ctx->rank = tp_rank;
    ctx->tp = tp_size;
    ctx->device = device;
    ctx->num_sms = prop.multiProcessorCount;
    ctx->h = c.hidden;
    ctx->stage = stage;
    ctx->n_stages = n_stages;
    // the reference's even split of layers over stages (PP degree divides the model)
    ctx->layer0 = int(int64_t(stage) * c.num_layers / n_stages);
    ctx->L = int(int64_t(stage + 1) * c.num_layers / n_stages) - ctx->layer0;
    ctx->hd = c.head_dim;
    ctx->nq_l = c.num_q_heads / tp_size;
    ctx->nkv_l = c.num_kv_heads / tp_size;
    ctx->G = ctx->nq_l / ctx->nkv_l;
    ctx->ffn_l = c.ffn / tp_size;
    ctx->vocab_l = c.vocab / tp_size;
    ctx->seed = weight_seed;
    ctx->grp = grp;
    ctx->tu = tuning_from_env();
    if (const char* f = getenv("SS_ATTN_SPLIT")) ctx->decode_split = std::max(64, atoi(f) / 64 * 64);  // dev tuning
    if (const char* f = getenv("SS_ATTN_FUSED_COMBINE")) ctx->fused_combine = atoi(f);
    if (const char* f = getenv("SS_ATTN_TC")) ctx->attn_tc = atoi(f);  // dev: 0 = mma.sync prefill tiles
    if (ctx->fused_combine) ctx->attn_tc = 0;  // the in-kernel split merge exists on the mma.sync path only
    if (const char* f = getenv("SS_KV_PF_MB")) ctx->kv_pf_mb = atoi(f);  // dev tuning
    if (const char* f = getenv("SS_FUSE_ROPE")) ctx->fuse_rope = atoi(f);
    if (const char* f = getenv("SS_GRAPHS")) ctx->graphs = atoi(f);  // dev A/B
    if (const char* f = getenv("SS_TP_ALLREDUCE")) ctx->ipc_algo = atoi(f);
    // every allocation below lands on `device`, whatever the calling thread's current device
    if (cudaSetDevice(device) != cudaSuccess) {
        delete ctx;
        return fail(nullptr, SS_CUDA_ERROR, "cudaSetDevice");
    }
    if (cudaMalloc(&ctx->sk_part, gemm_part_floats(ctx->num_sms) * 4) != cudaSuccess ||
        cudaMalloc(&ctx->sk_flags, 2 * gemm_flag_words(ctx->num_sms) * 4) != cudaSuccess ||
        cudaMemset(ctx->sk_flags, 0, 2 * gemm_flag_words(ctx->num_sms) * 4) != cudaSuccess ||
        cudaMalloc(&ctx->d_epoch, 4) != cudaSuccess || cudaMemset(ctx->d_epoch, 0, 4) != cudaSuccess) {
        std::string m = "stream-K workspace allocation";
        ss_destroy(ctx);
        return fail(nullptr, SS_OUT_OF_MEMORY, m);
    }
    auto bail = [&](ss_status s) {
        std::string m = ctx->err;
        ss_destroy(ctx);
        g_create_err = m;
        return s;
    };
    if (grp) ctx->st = grp->st;
    else if (cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(ctx, SS_CUDA_ERROR, "stream create"));
    cudaEventCreate(&ctx->ev0);
    cudaEventCreate(&ctx->ev1);
    cudaEventCreateWithFlags(&ctx->ev_stage, cudaEventDisableTiming);

    // ---- weights: one allocation
    const int64_t h = c.hidden, hd = c.head_dim;
    const int64_t qkv_rows = int64_t(ctx->nq_l + 2 * ctx->nkv_l) * hd, qd = int64_t(ctx->nq_l) * hd;
    const int64_t per_layer = qkv_rows * h + h * qd + 2 * int64_t(ctx->ffn_l) * h + h * ctx->ffn_l + 2 * h;
    const bool first = stage == 0, last = stage == n_stages - 1;
    size_t bytes = size_t(per_layer + 256 * 6) * 2 * size_t(ctx->L) +
                   size_t((first ? int64_t(c.vocab) * h : 0) + (last ? int64_t(ctx->vocab_l) * h + h : 0)) * 2 + 4096;
    if (cudaMalloc(&ctx->wmem, bytes) != cudaSuccess) return bail(fail(ctx, SS_OUT_OF_MEMORY, "weights allocation"));
    uint8_t* p = ctx->wmem;
    ctx->layers.resize(size_t(ctx->L));
    const float s_qkv = ss_weight_scale(SS_T_Q, h, c.num_layers);
    const float s_o = ss_weight_scale(SS_T_O, int64_t(c.num_q_heads) * hd, c.num_layers);
    const float s_gu = ss_weight_scale(SS_T_GATE, h, c.num_layers);
    const float s_dn = ss_weight_scale(SS_T_DOWN, c.ffn, c.num_layers);
    for (int ll = 0; ll < ctx->L; ++ll) {
        const int l = ctx->layer0 + ll;  // global layer index: the same synthetic weights on every stage split
        Layer& W = ctx->layers[size_t(ll)];
        W.wqkv = carve<bf16>(p, size_t(qkv_rows * h));
        W.wo = carve<bf16>(p, size_t(h * qd));
        W.wgu = carve<bf16>(p, size_t(2 * ctx->ffn_l * h));
        W.wdown = carve<bf16>(p, size_t(h * ctx->ffn_l));
        W.attn_norm = carve<bf16>(p, size_t(h));
        W.mlp_norm = carve<bf16>(p, size_t(h));
        ss_status s;
        if ((s = init_weight(ctx, W.wqkv, W_QKV, l, qkv_rows, h, s_qkv, s_qkv, s_qkv)) ||
            (s = init_weight(ctx, W.wo, W_O, l, h, qd, s_o, s_o, s_o)) ||
            (s = init_weight(ctx, W.wgu, W_GU, l, 2 * ctx->ffn_l, h, s_gu, s_gu, s_gu)) ||
            (s = init_weight(ctx, W.wdown, W_DOWN, l, h, ctx->ffn_l, s_dn, s_dn, s_dn)) ||
            (s = init_weight(ctx, W.attn_norm, W_NORM, l, 1, h, 1, 1, 1, SS_NORM_ATTN)) ||
            (s = init_weight(ctx, W.mlp_norm, W_NORM, l, 1, h, 1, 1, 1, SS_NORM_MLP)))
            return bail(s);
        // the pre-attention / pre-MLP RMSNorm gains are folded into the consuming
        // projections' K columns (the norm itself is folded into their epilogues)
        if (fold_gain_launch(W.wqkv, W.attn_norm, qkv_rows, h, ctx->st) != cudaSuccess ||
            fold_gain_launch(W.wgu, W.mlp_norm, 2 * ctx->ffn_l, h, ctx->st) != cudaSuccess)
            return bail(fail(ctx, SS_CUDA_ERROR, "norm-gain fold launch"));
        if (!bmaps(W.tb_qkv, W.wqkv, qkv_rows, h) || !bmaps(W.tb_o, W.wo, h, qd) ||
            !bmaps(W.tb_gu, W.wgu, 2 * ctx->ffn_l, h) || !bmaps(W.tb_down, W.wdown, h, ctx->ffn_l))
            return bail(fail(ctx, SS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (weights)"));
    }
    if (first) {
        ctx->embed = carve<bf16>(p, size_t(int64_t(c.vocab) * h));
        if (ss_status s = init_weight(ctx, ctx->embed, W_EMBED, 0, c.vocab, h, ss_embed_scale(), 0, 0)) return bail(s);
    }
    if (last) {
        ctx->lm_head = carve<bf16>(p, size_t(int64_t(ctx->vocab_l) * h));
        ctx->final_norm = carve<bf16>(p, size_t(h));
        ss_status s;
        if ((s = init_weight(ctx, ctx->lm_head, W_LMHEAD, 0, ctx->vocab_l, h, ss_weight_scale(-1, h, c.num_layers), 0,
                             0)) ||
            (s = init_weight(ctx, ctx->final_norm, W_NORM, 0, 1, h, 1, 1, 1, SS_NORM_FINAL)))
            return bail(s);
        if (!bmaps(ctx->tb_lm, ctx->lm_head, ctx->vocab_l, h))
            return bail(fail(ctx, SS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (lm head)"));
    }
    // ---- RoPE table (host, double precision; shared with the oracle via ss_synth.h)
    {
        const int half = c.head_dim / 2;
        std::vector<float2> tab(size_t(c.max_positions) * half);
        for (int64_t pp = 0; pp < c.max_positions; ++pp)
            for (int i = 0; i < half; ++i) {
                float cc, ss;
                ss_rope_cs(double(c.rope_theta), c.head_dim, pp, i, &cc, &ss);
                tab[size_t(pp) * half + i] = make_float2(cc, ss);
            }
        if (cudaMalloc(&ctx->rope, tab.size() * sizeof(float2)) != cudaSuccess)
            return bail(fail(ctx, SS_OUT_OF_MEMORY, "rope table"));
        cudaMemcpy(ctx->rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice);
    }
    // without an NCCL id a tp rank runs on the CUDA-IPC transport (ss_ipc_export / ss_ipc_open)
    if (tp_size > 1 && !grp && nccl_id) {
        std::string why;
        if (!g_nccl.load(why)) return bail(fail(ctx, SS_NCCL_ERROR, why));
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        ncclResult_t r = g_nccl.init_rank(&ctx->comm, tp_size, id, tp_rank);
        if (r != ncclSuccess) return bail(fail(ctx, SS_NCCL_ERROR, std::string("ncclCommInitRank: ") + g_nccl.err(r)));
    }
    if (cudaStreamSynchronize(ctx->st) != cudaSuccess)
        return bail(fail(ctx, SS_CUDA_ERROR, std::string("init: ") + cudaGetErrorString(cudaGetLastError())));
    *out = ctx;
    return SS_OK;
}

SS_API ss_status ss_create(const ss_model_cfg* cfg, int32_t tp_rank, int32_t tp_size, const void* nccl_id,
                           uint64_t weight_seed, int32_t device, ss_ctx** out) {
    return create_impl(cfg, tp_rank, tp_size, nccl_id, weight_seed, device, nullptr, out);
}

SS_API ss_status ss_create_pp_stage(const ss_model_cfg* cfg, int32_t stage, int32_t n_stages, uint64_t weight_seed,
                                    int32_t device, ss_ctx** out) {
    return create_impl(cfg, 0, 1, nullptr, weight_seed, device, nullptr, out, stage, n_stages);
}

SS_API ss_status ss_create_local_group(const ss_model_cfg* cfg, int32_t tp_size, uint64_t weight_seed,
                                       int32_t device, ss_ctx** out) {
    ss_ctx* ctx = nullptr;
    if (!cfg || !out || tp_size < 1 || tp_size > 8) return fail(ctx, SS_INVALID_ARG, "local group needs 1..8 ranks");
    LocalGroup* g = new LocalGroup();
    g->n = tp_size;
    g->live = 1;  // the creator's hold
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&g->st, cudaStreamNonBlocking) != cudaSuccess) {
        group_release(g);
        return fail(ctx, SS_CUDA_ERROR, "local group stream");
    }
    for (int r = 0; r < tp_size; ++r) {
        ++g->live;
        ss_ctx* c = nullptr;
        if (ss_status s = create_impl(cfg, r, tp_size, nullptr, weight_seed, device, g, &c)) {
            const std::string m = g_create_err;
            for (ss_ctx* done : g->ranks) ss_destroy(done);
            group_release(g);
            g_create_err = m;
            return s;
        }
        g->ranks.push_back(c);
        out[r] = c;
    }
    group_release(g);
    return SS_OK;
}

SS_API ss_status ss_forward_local_group(ss_ctx* const* ranks, int32_t n, const ss_batch_desc* desc, float* logits,
                                        int32_t* next, float* elapsed_ms) {
    ss_ctx* ctx = (ranks && n > 0) ? ranks[0] : nullptr;
    if (!ctx || !ctx->grp || n != ctx->grp->n) return fail(ctx, SS_INVALID_ARG, "not the full local TP group");
    LocalGroup* g = ctx->grp;
    for (int r = 0; r < n; ++r)
        if (!ranks[r] || ranks[r] != g->ranks[size_t(r)]) return fail(ctx, SS_INVALID_ARG, "ranks out of order");
    g->reset();
    CK(cudaSetDevice(ctx->device));
    CK(cudaEventRecord(ctx->ev0, g->st));
    std::vector<ss_status> st(size_t(n), SS_OK);
    auto body = [&](int r) {
        ss_ctx* c = ranks[r];
        cudaSetDevice(c->device);
        ss_status s = upload(c, desc, &c->scratch);
        if (s == SS_OK) s = enqueue_forward(c, &c->scratch);
        if (s != SS_OK) g->abort();
        st[size_t(r)] = s;
    };
    std::vector<std::thread> th;
    for (int r = 1; r < n; ++r) th.emplace_back(body, r);
    body(0);
    for (std::thread& t : th) t.join();
    for (int r = 0; r < n; ++r)
        if (st[size_t(r)] != SS_OK) {
            if (r != 0) ctx->err = "rank " + std::to_string(r) + ": " + ranks[r]->err;
            cudaStreamSynchronize(g->st);
            return st[size_t(r)];
        }
    CK(cudaEventRecord(ctx->ev1, g->st));
    if (ss_status s = read_outputs(ctx, &ctx->scratch, logits, next)) return s;
    CK(cudaEventSynchronize(ctx->ev1));
    if (elapsed_ms) CK(cudaEventElapsedTime(elapsed_ms, ctx->ev0, ctx->ev1));
    return SS_OK;
}

SS_API void ss_destroy(ss_ctx* ctx) {
    if (!ctx) return;
    DevGuard dg(ctx->device);
    if (ctx->st) cudaStreamSynchronize(ctx->st);
    if (ctx->comm) g_nccl.destroy(ctx->comm);
    for (int r = 0; r < kIpcMaxRanks; ++r)
        if (ctx->ipc_mapped[r]) cudaIpcCloseMemHandle(ctx->ipc_mapped[r]);
    if (ctx->ipc_region) cudaFree(ctx->ipc_region);
    cudaFree(ctx->dev_err);
    cudaFreeHost(ctx->host_err);
    cudaFree(ctx->wmem);
    cudaFree(ctx->rope);
    cudaFree(ctx->sk_part);
    cudaFree(ctx->sk_flags);
    cudaFree(ctx->d_epoch);
    graphs_clear(ctx);
    cudaFree(ctx->kc);
    cudaFree(ctx->vc);
    for (void* q : {(void*)ctx->x, (void*)ctx->xn, (void*)ctx->qkv, (void*)ctx->q, (void*)ctx->o, (void*)ctx->act,
                    (void*)ctx->part, (void*)ctx->xb, (void*)ctx->ssq, (void*)ctx->xo, (void*)ctx->logits_l, (void*)ctx->logits_g, (void*)ctx->logits,
                    (void*)ctx->next_tok, (void*)ctx->part_o, (void*)ctx->part_ml, (void*)ctx->comb_count, (void*)ctx->scratch.dev})
        cudaFree(q);
    cudaFreeHost(ctx->pinned);
    for (const Prof& p : ctx->pend) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (cudaEvent_t e : ctx->free_ev) cudaEventDestroy(e);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    cudaFree(ctx->part_red);
    cudaFree(ctx->chain_flags);
    cudaFree(ctx->chain_part);
    cudaFree(ctx->chain_trace);
    if (ctx->ev_stage) cudaEventDestroy(ctx->ev_stage);
    if (ctx->grp) {
        for (ss_ctx*& r : ctx->grp->ranks)
            if (r == ctx) r = nullptr;
        group_release(ctx->grp);
    } else if (ctx->st) {
        cudaStreamDestroy(ctx->st);
    }
    delete ctx;
}

SS_API ss_status ss_model_config(const ss_ctx* ctx, ss_model_cfg* out, int32_t* tp_rank, int32_t* tp_size) {
    if (!ctx || !out) return SS_INVALID_ARG;
    *out = ctx->cfg;
    if (tp_rank) *tp_rank = ctx->rank;
    if (tp_size) *tp_size = ctx->tp;
    return SS_OK;
}

SS_API ss_status ss_kv_alloc(ss_ctx* ctx, int64_t num_blocks, int32_t block_size) {
    if (!ctx || num_blocks < 1 || block_size != 16)
        return fail(ctx, SS_INVALID_ARG, "KV pool needs num_blocks >= 1 and block_size 16 (reference default)");
    DevGuard dg(ctx->device);
    cudaFree(ctx->kc);
    cudaFree(ctx->vc);
    ctx->kc = ctx->vc = nullptr;
    ctx->nblocks = 0;
    ctx->bs = block_size;
    ctx->layer_stride = num_blocks * ctx->nkv_l * block_size * ctx->hd;
    const size_t bytes = size_t(ctx->layer_stride) * ctx->L * 2;
    CK(cudaMalloc(&ctx->kc, bytes));
    CK(cudaMalloc(&ctx->vc, bytes));
    CK(cudaMemsetAsync(ctx->kc, 0, bytes, ctx->st));
    CK(cudaMemsetAsync(ctx->vc, 0, bytes, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    ctx->nblocks = num_blocks;
    ++ctx->ws_gen;
    return SS_OK;
}

SS_API ss_status ss_batch_upload(ss_ctx* ctx, const ss_batch_desc* desc, ss_batch** out) {
    if (!ctx || !out) return SS_INVALID_ARG;
    DevGuard dg(ctx->device);
    ss_batch* b = new ss_batch();
    if (ss_status s = upload(ctx, desc, b)) {
        cudaFree(b->dev);
        delete b;
        return s;
    }
    CK(cudaStreamSynchronize(ctx->st));
    *out = b;
    return SS_OK;
}

SS_API void ss_batch_free(ss_ctx* ctx, ss_batch* b) {
    if (!b) return;
    if (ctx) {
        DevGuard dg(ctx->device);
        cudaStreamSynchronize(ctx->st);
        if (ctx->last == b) ctx->last = nullptr;
    }
    cudaFree(b->dev);
    delete b;
}

SS_API ss_status ss_forward_enqueue(ss_ctx* ctx, const ss_batch* b) {
    if (!ctx || !b) return SS_INVALID_ARG;
    DevGuard dg(ctx->device);
    if (ss_status s = ensure_workspace(ctx, b->T, std::max(b->n_out, 1), b->part_rows)) return s;
    return run_forward(ctx, b);
}

// Pipeline hand-off: stage ctx (> 0) starts from the residual stream (fp32 x, its bf16 copy and
// the per-chunk sums of squares the first norm-folded QKV consumes) that stage prev left for the
// same batch; the copy runs on ctx's stream after prev's forward (event), over NVLink / peer
// memory when the stages are on different devices, and prev's stream then waits for the copy
// before its next forward may overwrite the buffers.
ss_status stage_handoff(ss_ctx* ctx, ss_ctx* prev, int T) {
    if (!prev || prev->stage != ctx->stage - 1 || prev->n_stages != ctx->n_stages || prev->h != ctx->h ||
        prev->T_cap < T)
        return fail(ctx, SS_INVALID_ARG, "pipeline stage s > 0 needs stage s - 1 of the same model and batch");
    CK(cudaStreamWaitEvent(ctx->st, prev->ev_stage, 0));
    const size_t h = size_t(ctx->h);
    CK(cudaMemcpyAsync(ctx->x, prev->x, size_t(T) * h * 4, cudaMemcpyDefault, ctx->st));
    CK(cudaMemcpyAsync(ctx->xb, prev->xb, size_t(T) * h * 2, cudaMemcpyDefault, ctx->st));
    CK(cudaMemcpyAsync(ctx->ssq, prev->ssq, size_t(T) * (h / 32) * 4, cudaMemcpyDefault, ctx->st));
    CK(cudaEventRecord(ctx->ev_stage, ctx->st));
    CK(cudaStreamWaitEvent(prev->st, ctx->ev_stage, 0));
    return SS_OK;
}

SS_API ss_status ss_forward_stage_enqueue(ss_ctx* ctx, const ss_batch* b, ss_ctx* prev) {
    if (!ctx || !b) return SS_INVALID_ARG;
    DevGuard dg(ctx->device);
    if ((ctx->stage == 0) != (prev == nullptr))
        return fail(ctx, SS_INVALID_ARG, "stage 0 takes no previous stage; every later stage needs stage - 1");
    if (ss_status s = ensure_workspace(ctx, b->T, std::max(b->n_out, 1), b->part_rows)) return s;
    if (prev)
        if (ss_status s = stage_handoff(ctx, prev, b->T)) return s;
    if (ss_status s = run_forward(ctx, b)) return s;
    CK(cudaEventRecord(ctx->ev_stage, ctx->st));
    return SS_OK;
}

SS_API ss_status ss_forward_pipeline(ss_ctx* const* stages, int32_t n, const ss_batch_desc* desc, float* logits,
                                     int32_t* next, float* stage_ms) {
    if (!stages || n < 1 || !desc) return fail(nullptr, SS_INVALID_ARG, "null argument");
    for (int i = 0; i < n; ++i)
        if (!stages[i] || stages[i]->stage != i || stages[i]->n_stages != n)
            return fail(stages[i], SS_INVALID_ARG, "stages[i] must be pipeline stage i of n");
    for (int i = 0; i < n; ++i) {  // every stage validates and uploads the same descriptor
        ss_ctx* c = stages[i];
        DevGuard dg(c->device);
        if (ss_status s = upload(c, desc, &c->scratch, i == 0 ? c->ev0 : nullptr)) return s;
    }
    for (int i = 0; i < n; ++i) {
        ss_ctx* ctx = stages[i];
        DevGuard dg(ctx->device);
        if (i > 0) {
            // this stage's own time starts at the hand-off, once the previous stage is done
            CK(cudaStreamWaitEvent(ctx->st, stages[i - 1]->ev_stage, 0));
            CK(cudaEventRecord(ctx->ev0, ctx->st));
            if (ss_status s = stage_handoff(ctx, stages[i - 1], ctx->scratch.T)) return s;
        }
        if (ss_status s = run_forward(ctx, &ctx->scratch)) return s;
        CK(cudaEventRecord(ctx->ev1, ctx->st));
        CK(cudaEventRecord(ctx->ev_stage, ctx->st));
    }
    ss_ctx* last = stages[n - 1];
    {
        DevGuard dg(last->device);
        if (ss_status s = read_outputs(last, &last->scratch, logits, next)) return s;
    }
    for (int i = 0; i < n; ++i) {
        ss_ctx* ctx = stages[i];
        DevGuard dg(ctx->device);
        CK(cudaEventSynchronize(ctx->ev1));
        if (stage_ms) CK(cudaEventElapsedTime(&stage_ms[i], ctx->ev0, ctx->ev1));
    }
    return SS_OK;
}

SS_API ss_status ss_read_outputs(ss_ctx* ctx, const ss_batch* b, float* logits, int32_t* next) {
    if (!ctx || !b) return SS_INVALID_ARG;
    DevGuard dg(ctx->device);
    return read_outputs(ctx, b, logits, next);
}

SS_API ss_status ss_forward_hybrid(ss_ctx* ctx, const ss_batch_desc* desc, float* logits, int32_t* next,
                                   float* elapsed_ms) {
    if (!ctx) return SS_INVALID_ARG;
    DevGuard dg(ctx->device);
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    if (ss_status s = upload(ctx, desc, &ctx->scratch, ctx->ev0)) return s;
    const auto t1 = clk::now();
    if (ss_status s = run_forward(ctx, &ctx->scratch)) return s;
    CK(cudaEventRecord(ctx->ev1, ctx->st));
    const auto t2 = clk::now();
    if (ss_status s = read_outputs(ctx, &ctx->scratch, logits, next)) return s;
    CK(cudaEventSynchronize(ctx->ev1));
    const auto t3 = clk::now();
    ctx->host_us[0] = std::chrono::duration<double, std::micro>(t1 - t0).count();
    ctx->host_us[1] = std::chrono::duration<double, std::micro>(t2 - t1).count();
    ctx->host_us[2] = std::chrono::duration<double, std::micro>(t3 - t2).count();
    if (elapsed_ms) CK(cudaEventElapsedTime(elapsed_ms, ctx->ev0, ctx->ev1));
    return SS_OK;
}

// Dev: host-side phases of the last ss_forward_hybrid (us): [0] validate + work list +
// staging (+ the H2D enqueue), [1] forward enqueue, [2] D2H + wait for the stream.
SS_API ss_status ss_debug_host_times(ss_ctx* ctx, double* out3) {
    if (!ctx || !out3) return SS_INVALID_ARG;
    for (int i = 0; i < 3; ++i) out3[i] = ctx->host_us[i];
    return SS_OK;
}

SS_API void* ss_stream(ss_ctx* ctx) { return ctx ? static_cast<void*>(ctx->st) : nullptr; }

SS_API ss_status ss_synchronize(ss_ctx* ctx) {
    if (!ctx) return SS_INVALID_ARG;
    DevGuard dg(ctx->device);
    if (ctx->ipc) CK(cudaMemcpyAsync(ctx->host_err, ctx->dev_err, 4, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return check_dev_err(ctx);
}

SS_API ss_status ss_kv_fill_synthetic(ss_ctx* ctx, const int32_t* block_table, int32_t n_blocks, int32_t rid,
                                      int32_t n_tokens, uint64_t seed) {
    if (!ctx || !block_table || n_tokens < 0 || int64_t(n_blocks) * ctx->bs < n_tokens)
        return fail(ctx, SS_INVALID_ARG, "bad synthetic fill arguments");
    DevGuard dg(ctx->device);
    for (int b = 0; b < n_blocks; ++b)
        if (block_table[b] < 0 || block_table[b] >= ctx->nblocks) return fail(ctx, SS_OUT_OF_KV, "block outside pool");
    int32_t* d = nullptr;
    CK(cudaMalloc(&d, size_t(std::max(n_blocks, 1)) * 4));
    CK(cudaMemcpy(d, block_table, size_t(n_blocks) * 4, cudaMemcpyHostToDevice));
    cudaError_t e = kv_fill_launch(ctx->kc, ctx->vc, ctx->layer_stride, ctx->L, d, n_tokens, rid, ctx->nkv_l,
                                   ctx->rank * ctx->nkv_l, ctx->cfg.num_kv_heads, ctx->hd, ctx->bs, seed, ctx->layer0,
                                   ctx->st);
    cudaError_t e2 = cudaStreamSynchronize(ctx->st);
    cudaFree(d);
    if (e != cudaSuccess || e2 != cudaSuccess) return fail(ctx, SS_CUDA_ERROR, "synthetic KV fill failed");
    return SS_OK;
}

SS_API ss_status ss_set_graphs(ss_ctx* ctx, int32_t enabled) {
    if (!ctx) return SS_INVALID_ARG;
    DevGuard dg(ctx->device);
    CK(cudaStreamSynchronize(ctx->st));
    ctx->graphs = enabled != 0;
    if (!ctx->graphs) graphs_clear(ctx);
    return SS_OK;
}

SS_API ss_status ss_set_tp_allreduce(ss_ctx* ctx, int32_t algo) {
    if (!ctx || algo < SS_AR_AUTO || algo > SS_AR_PUSH) return fail(ctx, SS_INVALID_ARG, "bad all-reduce algorithm");
    DevGuard dg(ctx->device);
    CK(cudaStreamSynchronize(ctx->st));
    ctx->ipc_algo = algo;
    graphs_clear(ctx);
    return SS_OK;
}

SS_API ss_status ss_graph_stats(ss_ctx* ctx, int64_t* captures, int64_t* replays) {
    if (!ctx) return SS_INVALID_ARG;
    if (captures) *captures = ctx->graph_captures;
    if (replays) *replays = ctx->graph_replays;
    return SS_OK;
}

SS_API ss_status ss_set_profiling(ss_ctx* ctx, int32_t enabled) {
    if (!ctx) return SS_INVALID_ARG;
    ctx->prof = enabled != 0;
    return SS_OK;
}

SS_API ss_status ss_kernel_times(ss_ctx* ctx, double* ms_out, int64_t* launches_out, int32_t reset) {
    if (!ctx) return SS_INVALID_ARG;
    DevGuard dg(ctx->device);
    CK(cudaStreamSynchronize(ctx->st));
    collect_prof(ctx);
    for (int k = 0; k < SS_K_NUM_CLASSES; ++k) {
        if (ms_out) ms_out[k] = ctx->ms[k];
        if (launches_out) launches_out[k] = ctx->launches[k];
        if (reset) {
            ctx->ms[k] = 0;
            ctx->launches[k] = 0;
        }
    }
    return SS_OK;
}

SS_API int64_t ss_launch_count(ss_ctx* ctx) { return ctx ? ctx->total_launches : 0; }

// ---------------------------------------------------------------- single kernels

SS_API ss_status ss_k_gemm(ss_ctx* ctx, const void* A, const void* B, void* D, int32_t M, int32_t N, int32_t K,
                           int32_t epi) {
    if (!ctx || epi < 0 || epi > 3) return fail(ctx, SS_INVALID_ARG, "bad gemm arguments");
    DevGuard dg(ctx->device);
    GemmPlan p;
    const int ldo = (epi == EPI_SWIGLU ? N / 2 : N) + ctx->tu.ldo_pad;  // dev: padded output rows
    if (!gemm_prepare(p, A, uint64_t(M), B, M, N, K, D, ldo, epi, ctx->num_sms, ctx->tu))
        return fail(ctx, SS_INVALID_ARG, "gemm shape unsupported (N%32, K%8, SwiGLU N%64) or tensor map failed");
    p.part = ctx->sk_part;
    p.flags = ctx->sk_flags + gemm_flag_words(ctx->num_sms);  // apart from the forward's flags
    p.epoch = ++ctx->sk_single_epoch;
    return launch(ctx, SS_K_GEMM_QKV, 1, [&] { return gemm_launch(p, ctx->st); });
}

SS_API ss_status ss_k_rmsnorm(ss_ctx* ctx, const float* x, const void* w, void* out, const int32_t* rows, int32_t M,
                              int32_t h, float eps) {
    if (!ctx || h % 8) return fail(ctx, SS_INVALID_ARG, "rmsnorm needs h % 8 == 0");
    DevGuard dg(ctx->device);
    return launch(ctx, SS_K_RMSNORM, 1, [&] {
        return rmsnorm_launch(x, static_cast<const bf16*>(w), static_cast<bf16*>(out), rows, M, h, eps, ctx->st);
    });
}

SS_API ss_status ss_k_rope_append(ss_ctx* ctx, const void* qkv, void* q_out, const int32_t* pos, const int64_t* slot,
                                  int32_t T, int32_t layer) {
    if (!ctx || layer < 0 || layer >= ctx->L || !ctx->kc) return fail(ctx, SS_INVALID_ARG, "bad rope/append args");
    DevGuard dg(ctx->device);
    return launch(ctx, SS_K_ROPE_APPEND, 1, [&] {
        return rope_append_launch(static_cast<const bf16*>(qkv), static_cast<bf16*>(q_out), pos, slot, ctx->rope, T,
                                  ctx->nq_l, ctx->nkv_l, ctx->hd, ctx->bs, ctx->kc + size_t(layer) * ctx->layer_stride,
                                  ctx->vc + size_t(layer) * ctx->layer_stride, ctx->st);
    });
}

SS_API ss_status ss_k_attention(ss_ctx* ctx, const ss_batch* b, const void* q, void* o, int32_t layer) {
    if (!ctx || !b || layer < 0 || layer >= ctx->L) return fail(ctx, SS_INVALID_ARG, "bad attention args");
    DevGuard dg(ctx->device);
    if (ss_status s = ensure_workspace(ctx, b->T, std::max(b->n_out, 1), b->part_rows)) return s;
    const AttnParams ap = attn_params(ctx, b, static_cast<const bf16*>(q), static_cast<bf16*>(o), layer);
    if (ss_status s = launch(ctx, SS_K_ATTN, 1, [&] { return attention_launch(ap, ctx->st); })) return s;
    if (b->n_combs && !ctx->fused_combine)
        return launch(ctx, SS_K_ATTN_COMBINE, 1, [&] { return attention_combine_launch(ap, ctx->st); });
    return SS_OK;
}

SS_API ss_status ss_kv_layer_ptrs(ss_ctx* ctx, int32_t layer, void** k, void** v) {
    if (!ctx || layer < 0 || layer >= ctx->L || !ctx->kc) return SS_INVALID_ARG;
    *k = ctx->kc + size_t(layer) * ctx->layer_stride;
    *v = ctx->vc + size_t(layer) * ctx->layer_stride;
    return SS_OK;
}

SS_API ss_status ss_weight_ptr(ss_ctx* ctx, const char* name, int32_t layer, void** ptr, int64_t* rows,
                               int64_t* cols) {
    if (!ctx || !name) return SS_INVALID_ARG;
    const std::string n(name);
    const int64_t h = ctx->h, qkv = int64_t(ctx->nq_l + 2 * ctx->nkv_l) * ctx->hd, qd = int64_t(ctx->nq_l) * ctx->hd;
    if ((n == "embed" && !ctx->embed) || ((n == "lm_head" || n == "final_norm") && !ctx->lm_head))
        return fail(ctx, SS_INVALID_ARG, "this pipeline stage holds no " + n);
    if (n == "embed") { *ptr = ctx->embed; *rows = ctx->cfg.vocab; *cols = h; return SS_OK; }
    if (n == "lm_head") { *ptr = ctx->lm_head; *rows = ctx->vocab_l; *cols = h; return SS_OK; }
    if (n == "final_norm") { *ptr = ctx->final_norm; *rows = 1; *cols = h; return SS_OK; }
    if (layer < 0 || layer >= ctx->L) return fail(ctx, SS_INVALID_ARG, "layer out of range");
    const Layer& W = ctx->layers[size_t(layer)];
    if (n == "wqkv") { *ptr = W.wqkv; *rows = qkv; *cols = h; return SS_OK; }
    if (n == "wo") { *ptr = W.wo; *rows = h; *cols = qd; return SS_OK; }
    if (n == "wgu") { *ptr = W.wgu; *rows = 2 * ctx->ffn_l; *cols = h; return SS_OK; }
    if (n == "wdown") { *ptr = W.wdown; *rows = h; *cols = ctx->ffn_l; return SS_OK; }
    if (n == "attn_norm") { *ptr = W.attn_norm; *rows = 1; *cols = h; return SS_OK; }
    if (n == "mlp_norm") { *ptr = W.mlp_norm; *rows = 1; *cols = h; return SS_OK; }
    return fail(ctx, SS_INVALID_ARG, "unknown weight name " + n);
}
