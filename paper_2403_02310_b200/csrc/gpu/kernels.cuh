// Launch interfaces of the sm_100a kernels (K1..K4) used by ctx.cu.
#pragma once
#include <cstdlib>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace ssk {

// ------------------------------------------------------------------ K3 GEMM
enum { EPI_BF16 = 0, EPI_RESADD = 1, EPI_SWIGLU = 2, EPI_F32 = 3, EPI_QKV = 4 };

// Extra epilogue operands (all optional / mode specific).
struct AttnItem;
struct EpiArgs {
    // RMSNorm folded into the consumer GEMM: A holds the un-normalised bf16 rows;
    // each output row is scaled by rsqrt(sum(ssq_in[row][0..ssq_in_n)) * inv_dim + eps)
    // (norm gains are folded into the weights). Fixed summation order: deterministic.
    const float* ssq_in = nullptr;
    int ssq_in_n = 0;
    float inv_dim = 0.f, eps = 0.f;
    // EPI_RESADD producer side: bf16 copy of the updated residual row and the
    // per-(row, 32-column chunk) sums of squares the next consumer needs
    __nv_bfloat16* xb_out = nullptr;
    float* ssq_out = nullptr;
    // EPI_QKV: RoPE (rotate-half) of q/k heads + paged KV append; q -> q_out
    const int32_t* pos = nullptr;
    const int64_t* slot = nullptr;
    const float2* rope = nullptr;
    __nv_bfloat16* q_out = nullptr;
    __nv_bfloat16* kc = nullptr;
    __nv_bfloat16* vc = nullptr;
    int nq = 0, nkv = 0, hd = 0, bs = 16;
    // EPI_QKV, whole-tile schedule: CTA pairs beyond the tile count warm L2 with the first
    // pf_pages K/V pages of this layer's decode attention items (the cache that the
    // attention launch after this GEMM streams first), while the GEMM runs
    const struct AttnItem* pf_items = nullptr;
    int pf_n = 0, pf_pages = 0, pf_max_blocks = 0;
    const int32_t* pf_bt = nullptr;
    const int32_t* pf_ctx_len = nullptr;
    int l2hint = 0;  // operand L2 priority bits: 1 A evict-last, 2 B evict-first
    // Stream-K flag epochs are GemmPlan::epoch + *epoch_base when set: the forward's epoch
    // base lives in device memory (advanced by the forward's first kernel, embed), so a
    // CUDA graph of the forward replays with fresh epochs. Null: GemmPlan::epoch as is.
    const uint32_t* epoch_base = nullptr;
    // EPI_BF16, TP push reduce-scatter (SS_AR_PUSH): instead of `out`, each 8-element unit u
    // of the row-major [M][ldo] partial is stored into its owner rank o = u / push_share,
    // straight into o's exchange buffer push[o] (peer memory over NVLink) at landing unit
    // push_rank * push_share + (u - o * push_share). push_n = 0: plain stores to `out`.
    __nv_bfloat16* push[8] = {};
    int push_n = 0, push_rank = 0;
    int64_t push_share = 0;
};

// Developer tuning overrides (the SS_* environment variables the scripts/ A/B sweeps set),
// read once per context at ss_create by tuning_from_env() and carried explicitly to the
// launchers; nothing on the launch path reads the environment. Defaults = production.
struct Tuning {
    int attn_tc_mode = -1;    // SS_ATTN_TC_MODE: force the tensor-core prefill flavour (1..3)
    int attn_order = 0;       // SS_ATTN_ORDER=1: prefill row tiles first in the work list
    int attn_l2hint = 1;      // SS_ATTN_L2HINT: K/V L2 priority bits (AttnParams::kv_hint)
    int attn_tc2_first = 0;   // SS_ATTN_TC2_FIRST: compact prefill launch before the decodes
    int attn_pf_pages = 0;    // SS_ATTN_PF_PAGES: AttnParams::kv_pf_pages
    int gemm_l2hint = 3;      // SS_GEMM_L2HINT: operand L2 priority bits (EpiArgs::l2hint)
    int gemm_sk = -1;         // SS_GEMM_SK: force the schedule mode
    int gemm_splits = 0;      // SS_GEMM_SPLITS: force the split count
    int gemm_bn = 0;          // SS_GEMM_BN
    int gemm_cg = 0;          // SS_GEMM_CG
    int gemm_ar128 = 0;       // SS_GEMM_AR128: no 32-row A stages for M <= 32
    int gemm_debug = 0;       // SS_GEMM_DEBUG: print each launch's schedule
    int gemm_force[5][3] = {{-1, 0, 1}, {-1, 0, 1}, {-1, 0, 1}, {-1, 0, 1}, {-1, 0, 1}};  // SS_GEMM_<QKV|O|GATEUP|DOWN|LMHEAD>=mode,bn[,splits]
    int ldo_pad = 0;          // SS_GEMM_LDO_PAD (ss_k_gemm only)
    int chain = 0;            // SS_CHAIN bits: the fused projection chain instead of separate launches,
                              // 1 for batches above 128 tokens (CTA pairs; measured slower on the
                              // canonical batch), 2 up to 128 (weight streaming)
    int chain_splits[4] = {0, 0, 0, 0};  // SS_CHAIN_S=o,gu,down,qkv: K splits per chain phase (0: auto)
    int chain_debug = 0;      // SS_CHAIN_DEBUG: print each chain launch
    int chain_trace = 0;      // SS_CHAIN_TRACE: record the chain's per-item timeline (ss_debug_chain_trace)
    int gemm_dsm = 1;         // SS_GEMM_DSM=0: split-K partials of decode-sized single-CTA tiles
                              // through global memory + flags instead of the cluster's shared memory
    int gemm_max_groups = 0;  // SS_GEMM_MAXG: at most this many CTA groups per GEMM launch (dev scaling probe)
    int gemm_mc = 0;          // SS_GEMM_MC=1: weight-tile multicast between the CTA pairs of 4-CTA
                              // clusters (measured neutral: only 66 such clusters are co-resident)
};
Tuning tuning_from_env();

struct GemmPlan {
    CUtensorMap tmA, tmB;  // 64-byte aligned members of a 64-aligned struct
    int M = 0, N = 0, K = 0;
    int row0 = 0;  // the GEMM covers rows [row0, row0 + M) of A, out and the epilogue operands
    void* out = nullptr;
    int ldo = 0;
    int epi = 0;
    int cg = 1;    // CTAs per MMA group (2: cta_group::2 pairs, 256-row tiles)
    int ar = 128;  // rows of A per stage (32: M <= 32 single-CTA tiles; tmA's box must match)
    int bn = 256;  // tile N; each CTA stages bn / cg rows of B (the B map's box rows)
    int num_sms = 148;
    // stream-K workspace: partial accumulators [groups][128 * cg][bn] fp32 and one
    // ready flag per (group, CTA, epilogue warp); epoch must be unique per launch
    float* part = nullptr;
    uint32_t* flags = nullptr;
    uint32_t epoch = 0;
    int sk_mode = -1;  // -1 auto, 0 whole tiles round-robin, 1 stream-K, 2 lockstep split-K,
                       // 3 M-lockstep stream-K (super-groups of num_mt CTA pairs)
    int splits = 1;    // K slices per tile for mode 2 (tiles * splits must fit one resident wave)
    int force_sk = -1, force_splits = 0, debug = 0;  // Tuning overrides applied at launch
    int max_groups = 0;  // > 0: at most this many CTA groups (SM budget of a concurrent launch)
    int dsm = 1;         // split-K over a thread-block cluster (see launch_t); 0: never
    int mc = 1;          // 2: clusters of two CTA pairs sharing weight tiles by TMA multicast
                         // (gemm_mc; tmB's box is then bn / cg / 2 rows)
    EpiArgs ea;
} __attribute__((aligned(64)));

// ---- Fused persistent chain of dependent projections (one launch per layer, TP = 1):
// O -> gate/up -> down -> next layer's QKV. Every CTA pair walks one global list of
// 256 x 256 tiles (phase-major; inside a phase column-tile-major, K slices, then M tiles),
// round-robin. A tile's TMA producer waits, per 64-column k-block of A, on the ready flag of
// the producing phase's output tile covering those columns, so a phase streams behind its
// predecessor instead of waiting for the whole grid, and a pair's next tile (from any phase)
// runs its main loop while its previous tile's epilogue drains (double-buffered TMEM): the
// per-launch fill, drain and wave-quantisation tails of separate launches disappear.
// K-split tiles publish fp32 partials; the last arriving split (per epilogue warp) sums all
// splits in fixed split order (deterministic) and runs the epilogue. All flags carry the
// launch epoch (epoch + *epoch_base), counters self-reset.
constexpr int kChainMaxPhases = 4;
struct ChainPhase {
    int N = 0, K = 0, epi = 0, splits = 1;
    int num_n = 0;       // 256-column tiles
    int item0 = 0;       // first global work item of the phase
    int dep = -1;        // phase whose output is this phase's A (-1: written before the launch)
    int res_dep = -1;    // phase whose residual-add output this phase's residual add reads
    int out_cols = 256;  // output columns per tile (SwiGLU: 128), for consumers' k-block mapping
    void* out = nullptr;
    int ldo = 0;
    uint32_t* ready = nullptr;  // [num_mt][num_n] tile-done flags (value = launch epoch)
    uint32_t* rcnt = nullptr;   // [num_mt][num_n] epilogue warps done (self-resetting)
    uint32_t* pcnt = nullptr;   // [num_mt][num_n][2][8] split arrivals per epilogue warp (self-resetting)
    float* part = nullptr;      // [num_mt][num_n][splits][cg][8 chunks][128][32] fp32 split partials
    EpiArgs ea;
};
struct ChainPlan {
    CUtensorMap tmA[kChainMaxPhases], tmB[kChainMaxPhases];  // A box ar x 64, B box (256 / cg) x 64
    int cg = 2;   // 2: CTA pairs, 256-row tiles; 1: single CTAs, 128-row tiles (decode-sized M)
    int ar = 128; // rows of A per stage (32: M <= 32)
    int n_phases = 0, M = 0, num_mt = 0, total_items = 0, num_sms = 148;
    uint32_t epoch = 0;
    const uint32_t* epoch_base = nullptr;
    int debug = 0;
    // dev timeline (SS_CHAIN_TRACE): per item, globaltimer ns at producer start / producer
    // done / MMA start / MMA done / epilogue start / epilogue done (leader CTA), or null
    unsigned long long* trace = nullptr;
    ChainPhase ph[kChainMaxPhases];
} __attribute__((aligned(64)));
// Items of one phase: num_mt * num_n * splits; fills item0 / total_items.
void gemm_chain_finalize(ChainPlan& p);
cudaError_t gemm_chain_launch(const ChainPlan& p, cudaStream_t st);

// Workspace sizes for gemm_launch (max over tile shapes) for num_sms SMs.
inline size_t gemm_part_floats(int num_sms) { return size_t(num_sms) * 128 * 256; }
inline size_t gemm_flag_words(int num_sms) { return size_t(num_sms) * 16; }

struct GemmShape {
    int cg, bn, splits, mode;  // mode: GemmPlan::sk_mode
    int ar = 128;              // GemmPlan::ar
};

bool make_tmap_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                  uint32_t box_cols);
// 2 when the picked shape shares weight tiles between the two M-tile pairs of a cluster by
// TMA multicast (CTA pairs, whole tiles or M-lockstep stream-K, even M-tile count), else 1.
int gemm_mc(const GemmShape& s, int M, const Tuning& tu);
// Tile shape for an M x N GEMM: minimises wave-quantised time over the compiled shapes.
GemmShape gemm_pick(int M, int N, int K, int epi, int num_sms, const Tuning& tu);
// A is [a_rows >= M][K] bf16; B is [N][K] bf16; out row stride ldo elements.
bool gemm_prepare(GemmPlan& p, const void* A, uint64_t a_rows, const void* B, int M, int N, int K, void* out,
                  int ldo, int epi, int num_sms, const Tuning& tu, int bn = 0);
cudaError_t gemm_launch(const GemmPlan& p, cudaStream_t st);

// ------------------------------------------------------------------ K1 attention
// One work item = (entry, kv head, row tile, key range). Rows of an entry for
// kv head h are (token j, head-in-group i) pairs, row = j * G + i.
struct AttnItem {
    int32_t entry;
    int32_t kv_head;
    int32_t row0;      // first row of the tile
    int32_t nrows;     // rows in the tile (<= 16: key-split decode mode; else tcgen05 <= 256 / mma.sync <= 64)
    int32_t key0;      // key range [key0, key1)
    int32_t key1;
    int32_t part;      // -1: final output; else partial slot base (rows)
    int32_t comb;      // split group (index into combines) or -1
};
struct AttnCombine {  // one split group: partial slots base + s * nrows_pad
    int32_t entry;
    int32_t kv_head;
    int32_t row0;
    int32_t nrows;
    int32_t nsplit;
    int32_t part;
    int32_t stride;  // rows between consecutive splits' partial slots
    int32_t pad;
};
struct AttnParams {
    const __nv_bfloat16* q;      // [T][nq_l][hd]
    __nv_bfloat16* o;            // [T][nq_l][hd]
    const __nv_bfloat16* kc;     // layer K cache [nblocks][nkv_l][bs][hd]
    const __nv_bfloat16* vc;
    const int32_t* cu_q;         // [E+1]
    const int32_t* ctx_len;      // [E]
    const int32_t* block_table;  // [E][max_blocks]
    int32_t max_blocks;
    const AttnItem* items;
    int32_t n_items;
    float* part_o;               // [slots][hd] fp32 (unnormalised)
    float* part_ml;              // [slots][2]   (running max in log2 units, sum)
    const AttnCombine* combines;
    int32_t n_combines;
    int32_t nq_l, nkv_l, group, head_dim, block_size;
    float scale_log2;            // softmax scale * log2(e)
    int64_t layer_row0;          // first row of this layer in the 2D [rows][hd] TMA view of the cache
    int32_t* comb_count;         // per split group: finished splits (zeroed, self-resetting)
    int32_t fused_combine;       // 1: last split merges in-kernel; 0: attention_combine launch
    int32_t tc;                  // prefill row tiles: 0 mma.sync (64 rows); tcgen05 1 paired (256), 2 compact
                                 // (128, beside the decodes), 3 deep (128)
    int32_t n_tc;                // items[0, n_tc) are the tcgen05 tiles (launched first)
    int32_t wait_at_end;         // set by attention_launch for the second of its two launches
    int32_t num_sms;
    int32_t kv_hint;             // L2 priority bits: 1 decode K/V evict-first, 2 prefill K/V evict-last
    int32_t tc2_first;           // Tuning::attn_tc2_first
    int32_t kv_pf_pages;         // decode items: cached K/V pages each CTA asks L2 for before its grid-
                                 // dependency wait (the CTAs PDL lands on SMs the QKV GEMM leaves idle)
};
// 2D TMA views [L * nblocks * nkv * 16][hd] of the K and V pools (box 16 x 64, SWIZZLE_128B).
cudaError_t attention_launch(const AttnParams& p, cudaStream_t st);
cudaError_t attention_combine_launch(const AttnParams& p, cudaStream_t st);

// ------------------------------------------------------------------ K2/K4 elementwise
// x = embed[tokens] (fp32) plus the bf16 copy and per-chunk sums of squares the
// first (norm-folded) QKV GEMM consumes.
// epoch_ctr (nullable): the forward's device epoch base, advanced by epoch_stride once the
// previous forward has completed (EpiArgs::epoch_base)
cudaError_t embed_launch(const int32_t* tokens, const __nv_bfloat16* table, float* x, __nv_bfloat16* xb, float* ssq,
                         int T, int h, uint32_t* epoch_ctr, uint32_t epoch_stride, cudaStream_t st);
cudaError_t rmsnorm_launch(const float* x, const __nv_bfloat16* w, __nv_bfloat16* out, const int32_t* rows, int M,
                           int h, float eps, cudaStream_t st);
// RoPE (rotate-half) of q and k heads + paged KV append of k and v.
cudaError_t rope_append_launch(const __nv_bfloat16* qkv, __nv_bfloat16* q_out, const int32_t* pos,
                               const int64_t* slot, const float2* rope_cs, int T, int nq_l, int nkv_l, int hd,
                               int bs, __nv_bfloat16* kc, __nv_bfloat16* vc, cudaStream_t st);
// CUDA-IPC tensor-parallel transport (one process per GPU, buffers mapped from every
// rank): per rank two bf16 exchange buffers [T_cap][h] (alternating per all-reduce, so a
// rank never overwrites a buffer a peer may still read), an fp32 logits shard buffer and
// a flag array [8] (flag r = last collective epoch rank r reached).
constexpr int kIpcMaxRanks = 8;
struct IpcPeers {
    const __nv_bfloat16* buf[kIpcMaxRanks][2];
    // two-shot all-reduce: rank r's reduced share of the sum (bf16 [T_cap][h], only the
    // elements rank r owns are written), read by every rank in the gather phase
    __nv_bfloat16* red[kIpcMaxRanks];
    const float* logits[kIpcMaxRanks];
    uint32_t* flags[kIpcMaxRanks];
    int n, rank;
    // A peer that does not reach a collective within timeout_ns is reported, not trapped:
    // the waiting CTAs store kDevErrPeerTimeout | peer << 8 into *err (this rank's device
    // error word, read by the host after the forward) and skip the collective's work.
    uint32_t* err;
    uint64_t timeout_ns;
    // collective epochs are the launch's epoch + *epoch_base (see EpiArgs::epoch_base)
    const uint32_t* epoch_base;
};
constexpr uint32_t kDevErrPeerTimeout = 1;
cudaError_t ipc_allreduce_residual_launch(float* x, const IpcPeers& pe, int slot, uint32_t epoch,
                                          __nv_bfloat16* xb, float* ssq, int T, int h, cudaStream_t st);
// Two-shot all-reduce (reduce-scatter + all-gather over peer memory), for tp >= 4 where
// the one-shot pull reads (tp - 1) full messages per rank: phase 1 sums this rank's
// 1/tp share of the elements over every rank's partial (fixed rank order, fp32) into its
// red buffer; phase 2 reads every rank's share and adds it to the residual (+ xb / ssq).
// Per-rank ingress 2 (tp - 1) / tp messages, the ring's figure. Each phase opens with a
// flag barrier (its own epoch).
cudaError_t ipc_reduce_scatter_launch(const IpcPeers& pe, int slot, uint32_t epoch, int T, int h, cudaStream_t st);
cudaError_t ipc_push_reduce_launch(const IpcPeers& pe, int slot, uint32_t epoch, int T, int h, cudaStream_t st);
cudaError_t ipc_gather_residual_launch(float* x, const IpcPeers& pe, uint32_t epoch, __nv_bfloat16* xb, float* ssq,
                                       int T, int h, cudaStream_t st);
cudaError_t ipc_gather_logits_launch(const IpcPeers& pe, uint32_t epoch, float* out, int rows, int vl,
                                     cudaStream_t st);
// x += part (TP all-reduce result), also refreshing xb / ssq for the next norm-folded GEMM.
cudaError_t residual_add_launch(float* x, const __nv_bfloat16* part, __nv_bfloat16* xb, float* ssq, int T, int h,
                                cudaStream_t st);
cudaError_t argmax_launch(const float* logits, int rows, int V, int ld, int32_t* out, cudaStream_t st);
// logits gathered [tp][rows][V_l] -> [rows][tp * V_l]
struct PeerBufs {
    const __nv_bfloat16* p[8];
};
// out = sum of n_src (<= 8) bf16 buffers of n elements (n % 8 == 0).
cudaError_t peer_sum_launch(__nv_bfloat16* out, const PeerBufs& src, int n_src, int64_t n, cudaStream_t st);
cudaError_t gather_vocab_launch(const float* in, float* out, int tp, int rows, int vl, cudaStream_t st);

// Synthetic initialisers (ss_synth.h).
enum WeightKind { W_QKV = 0, W_O = 1, W_GU = 2, W_DOWN = 3, W_EMBED = 4, W_LMHEAD = 5, W_NORM = 6 };
struct WeightInit {
    int kind, layer, rank;
    int64_t rows, cols;
    int nq_l, nkv_l, hd, ffn_l, vocab_l;
    uint64_t seed;
    float scale_a, scale_b, scale_c;  // per-tag scales (q/k/v or gate/up)
    int norm;                         // W_NORM: which gain (SS_NORM_*)
    // W_QKV, hd = 128: store each head's 32-row chunks as [0-31, 64-95, 32-63, 96-127], so
    // every rotate-half partner pair is two adjacent 32-column chunks of the QKV output (the
    // fused QKV epilogue then needs no whole-head tiles: any 64-column multiple works)
    int qkv_interleave;
};
cudaError_t init_weight_launch(__nv_bfloat16* w, const WeightInit& wi, cudaStream_t st);
// w[r][c] = bf16(w[r][c] * gain[c]): an RMSNorm gain folded into the consuming projection
// (x_hat * g) . W^T = x_hat . (W diag(g))^T.
cudaError_t fold_gain_launch(__nv_bfloat16* w, const __nv_bfloat16* gain, int64_t rows, int64_t cols, cudaStream_t st);
// layer0: global index of the pool's first layer (a pipeline stage holds layers layer0 ..).
cudaError_t kv_fill_launch(__nv_bfloat16* kbase, __nv_bfloat16* vbase, int64_t layer_stride, int L,
                           const int32_t* bt_dev, int n_tokens, int rid, int nkv_l, int kv_off, int nkv_g, int hd,
                           int bs, uint64_t seed, int layer0, cudaStream_t st);
// Advances the forward's device epoch base (what embed does on the first pipeline stage) for
// a later stage, whose forward starts from the previous stage's residual stream.
cudaError_t epoch_advance_launch(uint32_t* epoch_ctr, uint32_t epoch_stride, cudaStream_t st);

}  // namespace ssk

namespace ssk {
// Launch with the programmatic-stream-serialization attribute (PDL) and an
// optional cluster shape. Every kernel in this library calls pdl_wait() before
// its first global access, so PDL launches are always safe.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              int cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int n = 0;
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
    if (cluster_x > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = cluster_x;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace ssk
