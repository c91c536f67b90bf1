"""ctypes bindings of the two C ABIs (include/ss_host.h, include/ss_gpu.h).

The shared libraries are built in-tree by `make` (see __graft_entry__.build).
Loading fails loudly when they are missing: there is no Python or CPU
fallback for anything on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
GPU_SO = os.path.join(PKG_DIR, "libss_gpu.so")
HOST_SO = os.path.join(PKG_DIR, "libss_host.so")

(SS_OK, SS_INVALID_ARG, SS_OUT_OF_KV, SS_INFEASIBLE, SS_OUT_OF_MEMORY, SS_CUDA_ERROR, SS_NCCL_ERROR, SS_INTERNAL,
 SS_CALIBRATION) = range(9)


class SSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[ss status {status}] {msg}")
        self.status = status


class ContractViolation(SSError):
    """servesim::ContractViolation (reference core.hpp:18-20)."""


class OutOfKvBlocks(SSError):
    """servesim::OutOfKvBlocks (reference core.hpp:22-24)."""


class InfeasibleSlo(SSError):
    """servesim::InfeasibleSlo (reference core.hpp:26-28)."""


class CalibrationError(SSError):
    """servesim::CalibrationError (reference costmodel.hpp:74-76)."""


def raise_for(status: int, msg: str) -> None:
    if status == SS_OK:
        return
    cls = {SS_INVALID_ARG: ContractViolation, SS_OUT_OF_KV: OutOfKvBlocks, SS_INFEASIBLE: InfeasibleSlo,
           SS_CALIBRATION: CalibrationError}.get(status, SSError)
    raise cls(status, msg)


class ReplicaCfg(C.Structure):
    _fields_ = [
        ("scheduler", C.c_int32), ("token_budget", C.c_int32), ("max_batch_size", C.c_int32),
        ("max_num_batched_tokens", C.c_int32), ("max_batch_size_orca", C.c_int32),
        ("tp_degree", C.c_int32), ("pp_degree", C.c_int32), ("kv_blocks", C.c_int64),
        ("kv_block_size", C.c_int32), ("tile_size", C.c_int32), ("chunk_align", C.c_int32),
        ("reserve_decode_tokens", C.c_int32), ("kv_watermark_frac", C.c_double),
        ("pipeline_tbt_factor", C.c_double), ("hybrid_batching", C.c_int32),
    ]


class CostParams(C.Structure):
    _fields_ = [
        ("per_token_linear_ms", C.c_double), ("saturation_tokens", C.c_int32),
        ("attn_prefill_quad_ms", C.c_double), ("attn_kv_read_ms", C.c_double),
        ("attn_decode_per_kv_ms", C.c_double), ("fixed_overhead_ms", C.c_double),
        ("tp_comm_ms", C.c_double), ("pp_send_ms", C.c_double), ("tile_size", C.c_int32),
        ("tile_penalty_frac", C.c_double),
    ]


class CalibOpts(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("tile_penalty_frac", C.c_double), ("max_saturation_tokens", C.c_int32)]


class TraceRow(C.Structure):
    _fields_ = [("arrival_us", C.c_int64), ("prompt_tokens", C.c_int32), ("output_tokens", C.c_int32)]


class EntryRow(C.Structure):
    _fields_ = [("request_id", C.c_int32), ("kind", C.c_int32), ("chunk_tokens", C.c_int32), ("prefix_tokens", C.c_int64)]


class CapacityOpts(C.Structure):
    _fields_ = [("qps_low", C.c_double), ("max_qps", C.c_double), ("rel_width", C.c_double), ("parallel", C.c_int32)]


class AnchorRow(C.Structure):
    _fields_ = [("entries", C.POINTER(EntryRow)), ("n_entries", C.c_int32), ("observed_ms", C.c_double)]


class Latency(C.Structure):
    _fields_ = [
        ("ttft_median_ms", C.c_double), ("tbt_p99_ms", C.c_double), ("tbt_median_ms", C.c_double),
        ("sched_delay_median_ms", C.c_double), ("throughput_tps", C.c_double),
        ("bubble_fraction", C.c_double), ("makespan_ms", C.c_double), ("tbt_samples", C.c_int64),
        ("n_requests", C.c_int32),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class SimOpts(C.Structure):
    _fields_ = [("keep_events", C.c_int32), ("max_events", C.c_int64), ("gpu", C.c_void_p),
                ("token_seed", C.c_uint64), ("check_block_tables", C.c_int32),
                ("gpu_stages", C.c_void_p), ("n_gpu_stages", C.c_int32)]


class CapacityProbe(C.Structure):
    _fields_ = [("qps", C.c_double), ("pass_", C.c_int32), ("report", Latency)]


class ModelCfg(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int32), ("hidden", C.c_int32), ("num_q_heads", C.c_int32),
        ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32), ("vocab", C.c_int32),
        ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("max_positions", C.c_int32),
    ]


class BatchDesc(C.Structure):
    _fields_ = [
        ("num_entries", C.c_int32), ("num_tokens", C.c_int32), ("cu_q", C.POINTER(C.c_int32)),
        ("ctx_len", C.POINTER(C.c_int32)), ("pos", C.POINTER(C.c_int32)), ("token_ids", C.POINTER(C.c_int32)),
        ("slot", C.POINTER(C.c_int64)), ("block_table", C.POINTER(C.c_int32)), ("max_blocks", C.c_int32),
        ("out_rows", C.POINTER(C.c_int32)), ("n_out", C.c_int32),
    ]


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


_gpu = None
_host = None


def gpu_lib():
    global _gpu
    if _gpu is None:
        if not os.path.exists(GPU_SO):
            raise ImportError(f"{GPU_SO} missing: run `make` (or __graft_entry__.build()) first")
        lib = C.CDLL(GPU_SO)
        P, I32, I64, F = C.c_void_p, C.c_int32, C.c_int64, C.c_float
        _sig(lib, "ss_create", I32, [C.POINTER(ModelCfg), I32, I32, P, C.c_uint64, I32, C.POINTER(P)])
        _sig(lib, "ss_destroy", None, [P])
        _sig(lib, "ss_model_config", I32, [P, C.POINTER(ModelCfg), C.POINTER(I32), C.POINTER(I32)])
        _sig(lib, "ss_nccl_unique_id", I32, [P])
        _sig(lib, "ss_ipc_export", I32, [P, I32, P])
        _sig(lib, "ss_ipc_open", I32, [P, P])
        _sig(lib, "ss_kv_alloc", I32, [P, I64, I32])
        _sig(lib, "ss_forward_hybrid", I32, [P, C.POINTER(BatchDesc), P, P, C.POINTER(F)])
        _sig(lib, "ss_create_local_group", I32, [C.POINTER(ModelCfg), I32, C.c_uint64, I32, C.POINTER(P)])
        _sig(lib, "ss_forward_local_group", I32, [C.POINTER(P), I32, C.POINTER(BatchDesc), P, P, C.POINTER(F)])
        _sig(lib, "ss_create_pp_stage", I32, [C.POINTER(ModelCfg), I32, I32, C.c_uint64, I32, C.POINTER(P)])
        _sig(lib, "ss_forward_stage_enqueue", I32, [P, P, P])
        _sig(lib, "ss_forward_pipeline", I32, [C.POINTER(P), I32, C.POINTER(BatchDesc), P, P, P])
        _sig(lib, "ss_batch_upload", I32, [P, C.POINTER(BatchDesc), C.POINTER(P)])
        _sig(lib, "ss_forward_enqueue", I32, [P, P])
        _sig(lib, "ss_read_outputs", I32, [P, P, P, P])
        _sig(lib, "ss_batch_free", None, [P, P])
        _sig(lib, "ss_stream", P, [P])
        _sig(lib, "ss_synchronize", I32, [P])
        _sig(lib, "ss_kv_fill_synthetic", I32, [P, P, I32, I32, I32, C.c_uint64])
        _sig(lib, "ss_set_profiling", I32, [P, I32])
        _sig(lib, "ss_set_graphs", I32, [P, I32])
        _sig(lib, "ss_set_tp_allreduce", I32, [P, I32])
        _sig(lib, "ss_graph_stats", I32, [P, C.POINTER(I64), C.POINTER(I64)])
        _sig(lib, "ss_kernel_times", I32, [P, P, P, I32])
        _sig(lib, "ss_kernel_class_name", C.c_char_p, [I32])
        _sig(lib, "ss_launch_count", I64, [P])
        _sig(lib, "ss_last_error", C.c_char_p, [P])
        _sig(lib, "ss_k_gemm", I32, [P, P, P, P, I32, I32, I32, I32])
        _sig(lib, "ss_k_rmsnorm", I32, [P, P, P, P, P, I32, I32, F])
        _sig(lib, "ss_k_rope_append", I32, [P, P, P, P, P, I32, I32])
        _sig(lib, "ss_k_attention", I32, [P, P, P, P, I32])
        _sig(lib, "ss_kv_layer_ptrs", I32, [P, I32, C.POINTER(P), C.POINTER(P)])
        _sig(lib, "ss_weight_ptr", I32, [P, C.c_char_p, I32, C.POINTER(P), C.POINTER(I64), C.POINTER(I64)])
        _gpu = lib
    return _gpu


def host_lib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_SO):
            raise ImportError(f"{HOST_SO} missing: run `make` (or __graft_entry__.build()) first")
        lib = C.CDLL(HOST_SO)
        P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        _sig(lib, "ssh_replica_default", None, [C.POINTER(ReplicaCfg)])
        _sig(lib, "ssh_cost_preset", I32, [C.c_char_p, C.POINTER(CostParams)])
        _sig(lib, "ssh_make_trace", I32, [C.c_char_p, D, I32, C.c_uint64, C.POINTER(TraceRow)])
        _sig(lib, "ssh_make_trace_spec", I32, [D, D, D, D, I64, D, I32, C.c_uint64, C.POINTER(TraceRow)])
        _sig(lib, "ssh_simulate", I32, [C.POINTER(ReplicaCfg), C.POINTER(CostParams), C.POINTER(TraceRow), I32,
                                        C.POINTER(SimOpts), C.POINTER(P)])
        _sig(lib, "ssh_report_event_log", C.c_void_p, [P, C.POINTER(C.c_size_t)])
        _sig(lib, "ssh_report_summary", I32, [P, D, C.POINTER(Latency)])
        _sig(lib, "ssh_report_num_microbatches", I64, [P])
        _sig(lib, "ssh_report_microbatch", I32, [P, I64, C.POINTER(EntryRow), I32, C.POINTER(D), C.POINTER(I64)])
        _sig(lib, "ssh_report_peak_blocks", I64, [P])
        _sig(lib, "ssh_report_free", None, [P])
        _sig(lib, "ssh_iteration_time", D, [C.POINTER(EntryRow), I32, C.POINTER(CostParams), I32, I32])
        _sig(lib, "ssh_decode_reference_time", D, [C.POINTER(CostParams)])
        _sig(lib, "ssh_compute_token_budget", I32, [D, C.POINTER(CostParams), I32, C.POINTER(I32)])
        _sig(lib, "ssh_capacity_search", I32, [C.POINTER(ReplicaCfg), C.POINTER(CostParams), C.c_char_p, I32,
                                               C.c_uint64, D, C.POINTER(CapacityOpts), C.POINTER(SimOpts), C.POINTER(D),
                                               C.POINTER(I32), P, I32, C.POINTER(I32)])
        _sig(lib, "ssh_calibrate", I32, [C.POINTER(AnchorRow), I32, C.POINTER(CalibOpts), C.POINTER(CostParams),
                                         C.POINTER(D), C.POINTER(D), C.POINTER(D), C.POINTER(I32)])
        _sig(lib, "ssh_next_chunk_size", I32, [I32, I32, I32, I32, I32])
        _sig(lib, "ssh_percentile", I32, [C.POINTER(D), I64, D, C.POINTER(D)])
        _sig(lib, "ssh_desc_build", I32, [C.POINTER(EntryRow), I32, P, I32, I32, C.c_uint64, C.POINTER(P)])
        _sig(lib, "ssh_desc_canonical", I32, [I32, I32, I64, I64, I32, I32, C.c_uint64, C.POINTER(P)])
        _sig(lib, "ssh_desc_view", C.POINTER(BatchDesc), [P])
        _sig(lib, "ssh_desc_pool_blocks", I64, [P])
        _sig(lib, "ssh_desc_free", None, [P])
        _sig(lib, "ssh_session_create", I32, [I64, I32, I32, C.c_uint64, C.POINTER(P)])
        _sig(lib, "ssh_session_step", I32, [P, C.POINTER(EntryRow), I32, P, C.POINTER(P)])
        _sig(lib, "ssh_session_release", I32, [P, I32])
        _sig(lib, "ssh_session_peak_blocks", I64, [P])
        _sig(lib, "ssh_session_free", None, [P])
        _sig(lib, "ssh_last_error", C.c_char_p, [])
        _host = lib
    return _host


def host_check(status: int) -> None:
    if status != SS_OK:
        raise_for(status, host_lib().ssh_last_error().decode())


GPU_EXPORTS = [
    "ss_create", "ss_create_local_group", "ss_forward_local_group", "ss_create_pp_stage", "ss_forward_stage_enqueue",
    "ss_forward_pipeline", "ss_destroy", "ss_model_config", "ss_nccl_unique_id", "ss_ipc_export", "ss_ipc_open", "ss_kv_alloc", "ss_forward_hybrid",
    "ss_batch_upload", "ss_forward_enqueue", "ss_read_outputs", "ss_batch_free", "ss_stream", "ss_synchronize",
    "ss_set_graphs", "ss_graph_stats", "ss_set_tp_allreduce",
    "ss_kv_fill_synthetic", "ss_set_profiling", "ss_kernel_times", "ss_kernel_class_name", "ss_launch_count",
    "ss_last_error", "ss_k_gemm", "ss_k_rmsnorm", "ss_k_rope_append", "ss_k_attention", "ss_kv_layer_ptrs",
    "ss_weight_ptr",
]
HOST_EXPORTS = [
    "ssh_replica_default", "ssh_cost_preset", "ssh_make_trace", "ssh_make_trace_spec", "ssh_simulate",
    "ssh_report_event_log", "ssh_report_summary", "ssh_report_num_microbatches", "ssh_report_microbatch",
    "ssh_report_peak_blocks", "ssh_report_free", "ssh_iteration_time", "ssh_decode_reference_time",
    "ssh_compute_token_budget", "ssh_calibrate", "ssh_capacity_search", "ssh_next_chunk_size", "ssh_percentile", "ssh_desc_build", "ssh_desc_canonical",
    "ssh_desc_view", "ssh_desc_pool_blocks", "ssh_desc_free", "ssh_session_create", "ssh_session_step",
    "ssh_session_release", "ssh_session_peak_blocks", "ssh_session_free", "ssh_last_error",
]
