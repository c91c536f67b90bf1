/*
 * ss_gpu.h — the drop-in GPU boundary: one stall-free hybrid batch through a
 * Llama-style decoder on B200 (sm_100a), tensor-parallel over tp_size ranks.
 *
 * Replaces the reference's model step
 *     double iteration_time(const Batch&, const CostModelParams&, int tp, int pp)
 *     (reference proj/include/servesim/costmodel.hpp:60-61, called from
 *      Engine::try_issue, proj/src/engine.cpp:227)
 * with a real bf16 forward of the batch's T packed tokens. The measured device
 * time comes back in *elapsed_ms and goes through the same
 * max(1, llround(ms*1000)) conversion (engine.cpp:228, core.cpp:8).
 *
 * Batch composition (entry order = packed token order), token positions and
 * KV block tables are produced on the host by the restated scheduler
 * (ss_host.h); this library never makes scheduling decisions.
 *
 * Ownership: the caller owns every descriptor array for the duration of the
 * call (they are staged into pinned memory and copied to the device before the
 * call returns control on the stream). The library owns weights, the paged KV
 * pool and workspaces. Output buffers (logits, next tokens) are owned by the
 * caller. One ss_ctx per GPU rank, driven by one host thread; not reentrant.
 */
#ifndef SS_GPU_H
#define SS_GPU_H

#include <stddef.h>
#include <stdint.h>

#include "ss_status.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ss_ctx ss_ctx;

/* Model shape. The reference carries only hidden/ffn (presets.cpp:8-66); the
 * head geometry comes from the public model configs. */
typedef struct {
    int32_t num_layers;
    int32_t hidden;
    int32_t num_q_heads;  /* global */
    int32_t num_kv_heads; /* global */
    int32_t head_dim;
    int32_t ffn;          /* global intermediate size */
    int32_t vocab;
    float rope_theta;
    float rms_eps;
    int32_t max_positions; /* RoPE table length (>= longest prompt + output) */
} ss_model_cfg;

/* Descriptor of one hybrid batch (E entries, T packed tokens). Entry e owns
 * packed tokens [cu_q[e], cu_q[e+1]); token t sits at absolute position pos[t]
 * of its request and writes its K/V to paged slot slot[t] =
 * block_table[e][pos/bs]*bs + pos%bs. After the iteration the entry's KV
 * length is ctx_len[e] = prefix + chunk (engine.cpp:211-216). Logits are
 * produced for the packed rows listed in out_rows (every decode entry and every
 * chunk that completes its prompt, core.cpp:103-134). */
typedef struct {
    int32_t num_entries;
    int32_t num_tokens;
    const int32_t* cu_q;        /* [E+1] */
    const int32_t* ctx_len;     /* [E]   */
    const int32_t* pos;         /* [T]   */
    const int32_t* token_ids;   /* [T]   */
    const int64_t* slot;        /* [T]   */
    const int32_t* block_table; /* [E * max_blocks], -1 padded */
    int32_t max_blocks;
    const int32_t* out_rows;    /* [n_out] */
    int32_t n_out;
} ss_batch_desc;

/* Creates the per-rank context on `device`: allocates and initialises this
 * rank's weight shard from the counter-based generator (ss_synth.h), so every
 * rank and the CPU oracle see identical values. nccl_id is the 128-byte
 * ncclUniqueId from ss_nccl_unique_id on rank 0 (ignored when tp_size == 1). */
ss_status ss_create(const ss_model_cfg* cfg, int32_t tp_rank, int32_t tp_size,
                    const void* nccl_id, uint64_t weight_seed, int32_t device, ss_ctx** out);
void ss_destroy(ss_ctx* ctx);
ss_status ss_model_config(const ss_ctx* ctx, ss_model_cfg* out, int32_t* tp_rank, int32_t* tp_size);
ss_status ss_nccl_unique_id(void* out_128_bytes);

/* CUDA-IPC tensor-parallel transport, the alternative to NCCL (create the rank with
 * nccl_id = NULL): each rank exports its exchange region (two bf16 [max_tokens][hidden]
 * all-reduce buffers, an fp32 LM-head shard buffer, barrier flags) as a 64-byte
 * cudaIpcMemHandle_t, the caller all-gathers the handles (any out-of-band channel),
 * and every rank opens all of them (handles[r] = rank r's, rank order). The row-parallel
 * O / down projections then write their partials into the exchange buffer and one fused
 * kernel sums every rank's partial over peer memory (fixed rank order: identical on all
 * ranks) into the residual; the vocab shards are gathered the same way. */
ss_status ss_ipc_export(ss_ctx* ctx, int32_t max_tokens, void* handle_out_64_bytes);
ss_status ss_ipc_open(ss_ctx* ctx, const void* handles);

/* Paged KV pool: num_blocks blocks of block_size tokens for every layer and
 * this rank's KV heads. Layout per layer: [num_blocks][kv_heads_local] pages of
 * bs x hd bf16 for K and for V; inside a page, key r / dim d sits at
 * (d/64)*64*bs + r*64 + (((d%64)/8) ^ (r%8))*8 + d%8 (pre-swizzled, bs = 16). */
ss_status ss_kv_alloc(ss_ctx* ctx, int64_t num_blocks, int32_t block_size);

/* Synchronous forward of one hybrid batch from HOST descriptor arrays.
 * logits_out (nullable): [n_out][vocab] fp32. next_tokens_out (nullable):
 * [n_out] greedy argmax. elapsed_ms (nullable): device time of the forward. */
ss_status ss_forward_hybrid(ss_ctx* ctx, const ss_batch_desc* desc, float* logits_out,
                            int32_t* next_tokens_out, float* elapsed_ms);

/* Tensor parallelism on ONE device (validation transport where only one GPU is
 * visible): creates tp_size rank contexts (out[0..tp_size-1]) that share one
 * stream; ss_forward_local_group drives one host thread per rank through the
 * same sharded forward as a tp-GPU job, with every NCCL collective replaced by
 * host barriers + a peer-sum kernel (all-reduce) / peer copies (all-gather).
 * Each rank still needs ss_kv_alloc (+ fills) on its own context; outputs are
 * rank 0's. ss_destroy each context; the shared stream goes with the last. */
ss_status ss_create_local_group(const ss_model_cfg* cfg, int32_t tp_size, uint64_t weight_seed,
                                int32_t device, ss_ctx** out);
ss_status ss_forward_local_group(ss_ctx* const* ranks, int32_t n, const ss_batch_desc* desc,
                                 float* logits_out, int32_t* next_tokens_out, float* elapsed_ms);

/* Device-resident batches for steady-state timing: upload once, then enqueue
 * forwards on the context stream without host synchronisation. */
typedef struct ss_batch ss_batch;
ss_status ss_batch_upload(ss_ctx* ctx, const ss_batch_desc* desc, ss_batch** out);
ss_status ss_forward_enqueue(ss_ctx* ctx, const ss_batch* batch);
/* Copies the last enqueued forward's outputs to host (synchronises). */
ss_status ss_read_outputs(ss_ctx* ctx, const ss_batch* batch, float* logits_out,
                          int32_t* next_tokens_out);
void ss_batch_free(ss_ctx* ctx, ss_batch* batch);

/* Pipeline parallelism (reference engine.cpp:42-81, the stage model behind
 * iteration_time(..., pp) = t / pp, costmodel.cpp:55): a context holding stage
 * `stage` of `n_stages` of the model — layers [stage*L/n, (stage+1)*L/n), the
 * reference's even split; the embedding on stage 0, the final norm + LM head on
 * the last stage; the same synthetic weights and caches as the unpipelined model
 * (layers keep their global indices). tp_size 1. Each stage needs ss_kv_alloc
 * (its pool covers its own layers) and the same fills. Stages may sit on
 * different devices. */
ss_status ss_create_pp_stage(const ss_model_cfg* cfg, int32_t stage, int32_t n_stages,
                             uint64_t weight_seed, int32_t device, ss_ctx** out);
/* One stage of a forward of `batch` (uploaded on this stage's context).
 * prev = stage - 1 (NULL for stage 0): its residual stream for the batch is
 * handed over (device-to-device / peer copy ordered after prev's forward by an
 * event; prev's next forward waits for the copy). Outputs: ss_read_outputs on
 * the last stage. */
ss_status ss_forward_stage_enqueue(ss_ctx* ctx, const ss_batch* batch, ss_ctx* prev);
/* ss_forward_hybrid over a pipeline: stages[i] must be stage i of n. Uploads
 * the descriptor to every stage, runs the stages in order with the hand-offs,
 * reads the last stage's outputs; stage_ms (nullable, n entries): each stage's
 * device time, from its hand-off (stage 0: the descriptor upload) to its end. */
ss_status ss_forward_pipeline(ss_ctx* const* stages, int32_t n, const ss_batch_desc* desc,
                              float* logits_out, int32_t* next_tokens_out, float* stage_ms);

/* cudaStream_t of the context, for external event timing. */
void* ss_stream(ss_ctx* ctx);
ss_status ss_synchronize(ss_ctx* ctx);

/* CUDA graphs of the forward (default on). ss_forward_hybrid / ss_forward_enqueue capture
 * one graph per batch shape (token / entry / logit-row counts, attention work-list
 * counts, block-table width) the second time that shape is seen and replay it afterwards,
 * so a step costs one graph launch of host work instead of ~6 launches per layer. Off
 * while per-kernel profiling is on, for the one-device local group and on the NCCL
 * transport. Outputs are bitwise identical with and without graphs. */
ss_status ss_set_graphs(ss_ctx* ctx, int32_t enabled);
/* All-reduce algorithm of the CUDA-IPC TP transport (after O and down): SS_AR_ONESHOT pulls
 * every rank's partial (one barrier; (tp-1) messages of NVLink ingress per rank),
 * SS_AR_TWOSHOT reduce-scatters then all-gathers over peer memory (two barriers;
 * 2(tp-1)/tp messages per rank, the ring's byte count). SS_AR_PUSH is two-shot with the
 * reduce-scatter fused into the O / down GEMM epilogue: every output unit is stored straight
 * into its owner rank's exchange buffer (NVLink stores overlapping the remaining tiles), the
 * reduction then reads local memory; same bytes and bitwise the same result as SS_AR_TWOSHOT.
 * SS_AR_AUTO (default): push from tp >= 4 and a 1 MB message, else one-shot. All are
 * deterministic and identical on every rank. */
enum { SS_AR_AUTO = 0, SS_AR_ONESHOT = 1, SS_AR_TWOSHOT = 2, SS_AR_PUSH = 3 };
ss_status ss_set_tp_allreduce(ss_ctx* ctx, int32_t algo);
/* Graphs captured and replayed since creation (either pointer may be NULL). */
ss_status ss_graph_stats(ss_ctx* ctx, int64_t* captures, int64_t* replays);

/* Fills KV positions [0, n_tokens) of one request (given its block table)
 * with the synthetic cache values of ss_synth.h, for every layer. Used to
 * stand up canonical batches whose decodes sit at a 4k context. */
ss_status ss_kv_fill_synthetic(ss_ctx* ctx, const int32_t* block_table, int32_t n_blocks,
                               int32_t request_id, int32_t n_tokens, uint64_t kv_seed);

/* Per-kernel-class device time accounting (CUDA events around every launch on
 * the context stream). Classes: see ss_kernel_class_name. */
enum {
    SS_K_EMBED = 0,
    SS_K_RMSNORM = 1,
    SS_K_GEMM_QKV = 2,
    SS_K_ROPE_APPEND = 3,
    SS_K_ATTN = 4,
    SS_K_ATTN_COMBINE = 5,
    SS_K_GEMM_O = 6,
    SS_K_GEMM_GATEUP = 7,
    SS_K_GEMM_DOWN = 8,
    SS_K_ALLREDUCE = 9,
    SS_K_LMHEAD = 10,
    SS_K_ARGMAX = 11,
    SS_K_GEMM_CHAIN = 12, /* fused O -> gate/up -> down -> next QKV launch (TP = 1) */
    SS_K_NUM_CLASSES = 13
};
ss_status ss_set_profiling(ss_ctx* ctx, int32_t enabled);
/* ms_out/launches_out: SS_K_NUM_CLASSES entries accumulated since reset. */
ss_status ss_kernel_times(ss_ctx* ctx, double* ms_out, int64_t* launches_out, int32_t reset);
const char* ss_kernel_class_name(int32_t k);
/* Total kernel launches issued by this library on ctx since creation. */
int64_t ss_launch_count(ss_ctx* ctx);

const char* ss_last_error(ss_ctx* ctx); /* ctx may be NULL (creation errors) */

/* ---- single-kernel entry points (device pointers, ctx stream) ---------------
 * Used by the per-kernel parity tests; each is exactly the launch the fused
 * forward makes. */
/* K3: D[M,N] = A[M,K] . B[N,K]^T, bf16 in, fp32 accumulate (tcgen05/TMEM/TMA).
 * epilogue: 0 store bf16 D; 1 out_f32 += D; 2 SwiGLU over 32-column
 * gate/up interleave -> bf16 [M, N/2]; 3 store fp32 D. */
ss_status ss_k_gemm(ss_ctx* ctx, const void* A, const void* B, void* D, int32_t M, int32_t N,
                    int32_t K, int32_t epilogue);
/* K4: out_bf16[M,h] = rmsnorm(x_f32[M,h]) * w_bf16[h]; rows gathered through
 * row_idx when non-null. */
ss_status ss_k_rmsnorm(ss_ctx* ctx, const float* x, const void* w, void* out,
                       const int32_t* row_idx, int32_t M, int32_t h, float eps);
/* K2 (+K4 RoPE): rope q/k of qkv[T][(nq+2nkv)*hd] in place-free fashion,
 * q -> q_out[T][nq][hd], k/v -> paged cache of `layer` at slot[t]. Device
 * pointers for pos/slot. */
ss_status ss_k_rope_append(ss_ctx* ctx, const void* qkv, void* q_out, const int32_t* pos,
                           const int64_t* slot, int32_t T, int32_t layer);
/* K1: mixed paged attention for a device-resident batch of `layer`:
 * q[T][nq][hd] -> o[T][nq][hd]. */
ss_status ss_k_attention(ss_ctx* ctx, const ss_batch* batch, const void* q, void* o,
                         int32_t layer);
/* Reads back / writes raw KV of one layer ([num_blocks][kvh] pre-swizzled
 * pages, see ss_kv_alloc; bf16 each for K and V) for tests. */
ss_status ss_kv_layer_ptrs(ss_ctx* ctx, int32_t layer, void** k_ptr, void** v_ptr);
/* Device pointer of a weight tensor of this rank's shard: name in {"wqkv",
 * "wo", "wgu", "wdown", "attn_norm", "mlp_norm", "final_norm", "embed",
 * "lm_head"}; layer ignored for the global ones. rows/cols describe its
 * [rows][cols] bf16 layout. */
ss_status ss_weight_ptr(ss_ctx* ctx, const char* name, int32_t layer, void** ptr, int64_t* rows,
                        int64_t* cols);

#ifdef __cplusplus
}
#endif
#endif /* SS_GPU_H */
