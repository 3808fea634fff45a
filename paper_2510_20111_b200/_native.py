"""ctypes binding of libhzp_b200.so (the C-ABI in include/hzp_b200.h).

The product path has no fallback: if the shared library is missing or fails
to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HZP_B200_LIB", os.path.join(HERE, "libhzp_b200.so"))

# ---- status codes (hzp_b200.h) ----------------------------------------------
HZP_OK = 0
ERR_NON_DIVISIBLE, ERR_EMPTY_MODEL, ERR_BAD_FIELD = 1, 2, 3
ERR_SHAPE_MISMATCH, ERR_DTYPE_UNSUPPORTED = 4, 5
ERR_INVALID_POLICY, ERR_DEADLOCK = 6, 7
ERR_MEMORY, ERR_EQUIVALENCE, ERR_CUDA, ERR_ARG = 8, 9, 10, 11


class hzp_parallel(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("dp", "z1", "z2", "z3", "pp", "vpp", "cp", "tp")]


class hzp_model_spec(C.Structure):
    _fields_ = [("num_layers", C.c_int64), ("params_per_layer", C.c_int64),
                ("embedding_params", C.c_int64), ("seq_len", C.c_int64),
                ("micro_batch_size", C.c_int64), ("num_microbatches", C.c_int64),
                ("flops_per_token_per_layer", C.c_double), ("hidden_size", C.c_int64)]


class hzp_cost(C.Structure):
    _fields_ = [("num_nodes", C.c_int), ("ranks_per_node", C.c_int), ("intra_bw", C.c_double),
                ("inter_bw", C.c_double), ("intra_latency", C.c_double),
                ("inter_latency", C.c_double), ("device_flops", C.c_double)]


class hzp_task(C.Structure):
    _fields_ = [("id", C.c_int), ("kind", C.c_int), ("layer", C.c_int), ("microbatch", C.c_int),
                ("virtual_stage", C.c_int), ("pass_", C.c_int), ("duration", C.c_double),
                ("bytes", C.c_int64), ("num_deps", C.c_int), ("deps", C.POINTER(C.c_int))]


class hzp_reuse_report(C.Structure):
    _fields_ = [("r1_eliminated_ag", C.c_int), ("r2_merged_rs", C.c_int), ("r3_eliminated_ag", C.c_int),
                ("extra_cached_bytes", C.c_int64)]


class hzp_pool(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("slot_count", C.c_int), ("slot_bytes", C.c_int64)]


class hzp_sim_summary(C.Structure):
    _fields_ = [("makespan", C.c_double), ("compute_idle", C.c_double),
                ("compute_busy", C.c_double)]


class hzp_ledger(C.Structure):
    _fields_ = [("params_bf16", C.c_int64), ("grads_fp32", C.c_int64), ("replica_fp32", C.c_int64),
                ("momentum_fp32", C.c_int64), ("variance_fp32", C.c_int64), ("total_static", C.c_int64)]


class hzp_memory_report(C.Structure):
    _fields_ = [("peak_bytes", C.c_int64), ("fragmentation", C.c_double),
                ("peak_grad_buffer_bytes", C.c_int64), ("peak_memory", C.c_int64),
                ("makespan", C.c_double), ("n_samples", C.c_int)]


class hzp_plan_entry(C.Structure):
    _fields_ = [("id", C.c_int), ("kind", C.c_int), ("layer", C.c_int), ("microbatch", C.c_int),
                ("stream", C.c_int), ("slot", C.c_int), ("ring_wait", C.c_int),
                ("num_waits", C.c_int), ("waits", C.POINTER(C.c_int))]


class hzp_comm_tile(C.Structure):
    _fields_ = [("a_off", C.c_int64), ("b_off", C.c_int64), ("c_off", C.c_int64),
                ("mask", C.c_uint64), ("len", C.c_int32), ("local", C.c_int16),
                ("src", C.c_int16), ("vec", C.c_int32), ("pad_", C.c_int32)]


class hzp_engine_config(C.Structure):
    _fields_ = [("model", C.c_int), ("precision", C.c_int), ("num_dims", C.c_int),
                ("dims", C.c_int * 32), ("gpt_layers", C.c_int), ("gpt_hidden", C.c_int),
                ("gpt_heads", C.c_int), ("gpt_ffn", C.c_int), ("gpt_vocab", C.c_int),
                ("gpt_seq", C.c_int), ("batch", C.c_int), ("num_microbatches", C.c_int),
                ("par", hzp_parallel), ("prelaunch_depth", C.c_int), ("rs_slots", C.c_int),
                ("wgrad_slots", C.c_int), ("mode", C.c_int), ("lr", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("grad_scale", C.c_double), ("device", C.c_int), ("my_rank", C.c_int),
                ("timeline", C.c_int), ("gpt_experts", C.c_int), ("gpt_topk", C.c_int),
                ("gpt_capacity", C.c_int), ("reuse", C.c_int),
                ("recompute", C.c_int), ("gpt_swiglu", C.c_int)]


class hzp_launch_rec(C.Structure):
    _fields_ = [("task_id", C.c_int), ("kind", C.c_int), ("layer", C.c_int),
                ("microbatch", C.c_int), ("stream", C.c_int), ("slot", C.c_int),
                ("covered_first", C.c_int), ("covered_last", C.c_int)]


# (name, restype, argtypes) of every exported symbol — tests check the library
# exports exactly what include/hzp_b200.h declares.
_P = C.POINTER
_vp = C.c_void_p
SIGNATURES = [
    ("hzp_last_error", C.c_char_p, []),
    ("hzp_version", C.c_char_p, []),
    ("hzp_shard_elems", C.c_int64, [C.c_int64, C.c_int64]),
    ("hzp_validate", C.c_int, [_P(hzp_model_spec), _P(hzp_parallel), _P(hzp_cost)]),
    ("hzp_groups", C.c_int, [_P(hzp_parallel), C.c_int, _P(C.c_int), C.c_int, _P(C.c_int), _P(C.c_int)]),
    ("hzp_graph_build", C.c_int, [_P(hzp_model_spec), _P(hzp_parallel), _P(hzp_cost), C.c_int,
                                  C.c_int, _P(_vp)]),
    ("hzp_graph_build_pipeline", C.c_int, [_P(hzp_model_spec), _P(hzp_parallel), _P(hzp_cost), C.c_int,
                                           C.c_int, C.c_int, C.c_int, _P(hzp_reuse_report), _P(_vp)]),
    ("hzp_graph_destroy", None, [_vp]),
    ("hzp_graph_size", C.c_int, [_vp]),
    ("hzp_graph_task", C.c_int, [_vp, C.c_int, _P(hzp_task)]),
    ("hzp_graph_ag_slot_bytes", C.c_int64, [_vp]),
    ("hzp_graph_grad_buf_bytes", C.c_int64, [_vp]),
    ("hzp_derive_prelaunch_depth", C.c_int, [_vp, C.c_int64]),
    ("hzp_make_pools", C.c_int, [_vp, C.c_int, C.c_int, _P(hzp_pool), _P(hzp_pool)]),
    ("hzp_simulate", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _P(C.c_double), _P(C.c_double),
                               _P(hzp_sim_summary)]),
    ("hzp_memory_ledger", C.c_int, [_P(hzp_model_spec), _P(hzp_parallel), _P(hzp_ledger)]),
    ("hzp_memory_trace", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _P(C.c_double), _P(C.c_double), C.c_int64,
                                   _P(hzp_memory_report), _P(C.c_double), _P(C.c_int64), C.c_int]),
    ("hzp_utilization_report", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _P(C.c_double), _P(C.c_double),
                                         C.c_double, _P(C.c_double)]),
    ("hzp_plan_entry_get", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _P(hzp_plan_entry)]),
    ("hzp_comm_tiles", C.c_int, [_P(hzp_parallel), C.c_int64, _P(C.c_int64), _P(C.c_int64), C.c_int,
                                 C.c_int, C.c_int, _P(hzp_comm_tile), C.c_int, _P(C.c_int),
                                 _P(C.c_int), _P(C.c_int), _P(C.c_int), _P(C.c_int)]),
    ("hzp_ctx_create", C.c_int, [_P(hzp_engine_config), _P(_vp)]),
    ("hzp_ctx_destroy", None, [_vp]),
    ("hzp_ctx_layout", C.c_int, [_vp, _P(C.c_int64), _P(C.c_int64), _P(C.c_int64), _P(C.c_int64),
                                 _P(C.c_int)]),
    ("hzp_ctx_layer_range", C.c_int, [_vp, C.c_int, _P(C.c_int64), _P(C.c_int64)]),
    ("hzp_ctx_ipc_handle", C.c_int, [_vp, _vp, _P(C.c_size_t)]),
    ("hzp_ctx_open_peers", C.c_int, [_vp, _vp, C.c_size_t, C.c_int]),
    ("hzp_state_upload", C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int64]),
    ("hzp_state_download", C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int64]),
    ("hzp_state_set_step", C.c_int, [_vp, C.c_int, C.c_int]),
    ("hzp_state_get_step", C.c_int, [_vp, C.c_int, _P(C.c_int)]),
    ("hzp_state_init_random", C.c_int, [_vp, C.c_uint64, C.c_double]),
    ("hzp_step", C.c_int, [_vp, _vp, C.c_int, _P(C.c_float)]),
    ("hzp_sync", C.c_int, [_vp]),
    ("hzp_launch_log", C.c_int, [_vp, _P(hzp_launch_rec), C.c_int, _P(C.c_int)]),
    ("hzp_timeline", C.c_int, [_vp, _P(C.c_double), _P(C.c_double), C.c_int, _P(C.c_int),
                               _P(C.c_double), _P(C.c_double), _P(C.c_double)]),
    ("hzp_z1_timeline", C.c_int, [_vp, _P(C.c_double), _P(C.c_double), _P(C.c_double), C.c_int, _P(C.c_int)]),
    ("hzp_set_timeline", C.c_int, [_vp, C.c_int]),
    ("hzp_ctx_launch_count", C.c_int, [_vp, _P(C.c_int64)]),
    ("hzp_kernel_launches", C.c_uint64, []),
    ("hzp_ctx_stream", C.c_int, [_vp, C.c_int, _P(_vp)]),
    ("hzp_gemm_profile", C.c_int, [C.c_int]),
    ("hzp_gemm_profile_read", C.c_int, [_P(C.c_double), _P(C.c_double), _P(C.c_int)]),
    ("hzp_gemm_profile_dump", C.c_int, [_P(C.c_double), _P(C.c_double), _P(C.c_int), C.c_char_p, C.c_int]),
    ("hzp_gemm_profile_read_busy", C.c_int, [_P(C.c_double), _P(C.c_double), _P(C.c_double), _P(C.c_int)]),
    ("hzp_gemm_profile_dump_ex", C.c_int, [_P(C.c_double), _P(C.c_double), _P(C.c_double), _P(C.c_int),
                                           C.c_char_p, C.c_int]),
    ("hzp_ag_layer", C.c_int, [_vp, C.c_int, C.c_int]),
    ("hzp_ag_slot_download", C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int64]),
    ("hzp_wgrad_upload", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _P(C.c_float), C.c_int64]),
    ("hzp_rs_layer", C.c_int, [_vp, C.c_int, C.c_int]),
    ("hzp_collective_time", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _P(C.c_double)]),
    ("hzp_seeded_span", C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_double, _P(C.c_float)]),
    ("hzp_state_init_seeded", C.c_int, [_vp, C.c_uint64, C.c_double]),
    ("hzp_make_tokens", C.c_int, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int, _P(C.c_int32)]),
    ("hzp_z1_adam_step", C.c_int, [_vp]),
    ("hzp_zero_grads", C.c_int, [_vp]),
    ("hzp_barrier", C.c_int, [_vp]),
    ("hzp_gemm_bf16", C.c_int, [_vp, _vp, _vp] + [C.c_int] * 9 + [_vp]),
    ("hzp_gemm_bf16_ex", C.c_int, [_vp, _vp, _vp] + [C.c_int] * 11 + [_vp, _vp, C.c_int, _vp, C.c_int,
                                                                    _vp, C.c_float, _vp]),
    ("hzp_attention_fwd", C.c_int, [_vp, _vp, _vp] + [C.c_int] * 4 + [_vp]),
    ("hzp_attention_bwd", C.c_int, [_vp] * 7 + [C.c_int] * 4 + [_vp]),
    ("hzp_gemm_f32", C.c_int, [_vp, _vp, _vp] + [C.c_int] * 9 + [_vp]),
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not built — run `make -C paper_2510_20111_b200/csrc` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class HzpError(RuntimeError):
    """Base of the errors raised from HZP_ERR_* status codes."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ValidationError(HzpError):
    """ValidationError (include/hzp/config.hpp:68-77)."""


class CollectiveError(HzpError):
    """CollectiveError (include/hzp/collective.hpp:18-27)."""


class SchedError(HzpError):
    """SchedError (include/hzp/sched.hpp:55-64)."""


class CudaError(HzpError):
    pass


def check(rc: int) -> None:
    if rc == HZP_OK:
        return
    msg = (lib.hzp_last_error() or b"").decode(errors="replace")
    if rc in (ERR_NON_DIVISIBLE, ERR_EMPTY_MODEL, ERR_BAD_FIELD):
        raise ValidationError(rc, msg)
    if rc in (ERR_SHAPE_MISMATCH, ERR_DTYPE_UNSUPPORTED):
        raise CollectiveError(rc, msg)
    if rc in (ERR_INVALID_POLICY, ERR_DEADLOCK):
        raise SchedError(rc, msg)
    if rc == ERR_CUDA:
        raise CudaError(rc, msg)
    raise HzpError(rc, msg)
