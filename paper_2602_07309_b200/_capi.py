"""ctypes binding of the C-ABI in include/semrank_b200.h.

The shared library is built in-tree (paper_2602_07309_b200/lib/) by
``__graft_entry__.build()``. Importing this module fails loudly if it is
missing: there is no Python or CPU fallback for the scoring path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SEMRANK_LIB selects an alternative in-tree build (kernel tuning variants).
LIB_PATH = os.environ.get("SEMRANK_LIB") or os.path.join(_HERE, "lib", "libsemrank_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        " (the ranker has no CPU fallback)")

lib = C.CDLL(LIB_PATH)

# The structs below mirror include/semrank_b200.h at this ABI version; a
# stale build with other layouts would corrupt memory, so refuse it.
ABI_VERSION = 2
lib.sr_abi_version.restype = C.c_int32
if lib.sr_abi_version() != ABI_VERSION:
    raise ImportError(f"{LIB_PATH} has C-ABI version {lib.sr_abi_version()}, this binding needs "
                      f"{ABI_VERSION}: rebuild it with `python -c 'import __graft_entry__ as g; g.build()'`")

i32, i64, u64, f32, f64, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_size_t
P = C.POINTER


class ModelConfigC(C.Structure):
    _fields_ = [("n_layers", i32), ("d_model", i32), ("n_heads", i32), ("d_ff", i32),
                ("vocab_size", i32), ("max_seq", i32), ("yes_token_id", i32),
                ("no_token_id", i32), ("n_task_heads", i32),
                ("head_names", P(C.c_char_p)), ("head_arity", P(i32))]


class FlopReportC(C.Structure):
    _fields_ = [("attention_units", f64), ("linear_units", f64), ("t_q", f64),
                ("t_i_mean", f64), ("n_items", f64)]


class RequestC(C.Structure):
    _fields_ = [("prefix_tokens", P(i32)), ("t_q", i32), ("n_items", i32),
                ("item_offsets", P(i32)), ("item_tokens", P(i32)), ("item_rows", P(f32)),
                ("item_ids", P(i64)), ("mode", i32)]


class ResultC(C.Structure):
    _fields_ = [("scores", P(f64)), ("k", i32), ("topk_ids", P(i64)), ("topk_scores", P(f64)),
                ("topk_index", P(i32)), ("flops", FlopReportC),
                ("kv_incremental_per_item", f64), ("k_returned", i32)]


def _sig(name, res, *args):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = list(args)
    return fn


vp = C.c_void_p
_sig("sr_last_error", C.c_char_p)
_sig("sr_status_name", C.c_char_p, i32)
_sig("sr_abi_version", i32)
_sig("sr_config_validate", i32, P(ModelConfigC))
_sig("sr_config_default_toy", None, P(ModelConfigC))
_sig("sr_task_count", i32, P(ModelConfigC))
_sig("sr_weights_init", i32, P(ModelConfigC), u64, i32, P(vp))
_sig("sr_weights_load", i32, C.c_char_p, P(vp))
_sig("sr_weights_save", i32, vp, C.c_char_p)
_sig("sr_weights_from_tensors", i32, P(ModelConfigC), C.c_char_p, P(P(f32)), P(vp))
_sig("sr_weights_free", None, vp)
_sig("sr_weights_config", i32, vp, P(ModelConfigC))
_sig("sr_weights_version", C.c_char_p, vp)
_sig("sr_weights_tensor_count", sz, vp)
_sig("sr_weights_tensor", i32, vp, sz, P(C.c_char_p), P(P(f32)), P(sz))
_sig("sr_flops", i32, i32, i64, i64, i64, P(FlopReportC))
_sig("sr_multi_item_pair_count", i32, i32, P(i32), i32, P(i64))
_sig("sr_multi_item_mask", i32, i32, P(i32), i32, P(i32), i32, P(i32))
_sig("sr_plan_batches", i32, i32, P(i32), P(i32), P(i32), i64, P(i32), i32, P(i32), P(i64),
     i32, P(i32))
_sig("sr_request_report", i32, P(ModelConfigC), P(RequestC), P(FlopReportC), P(f64))
_sig("sr_topk_host", i32, P(f64), P(i64), i32, i32, P(i64), P(f64), P(i32))
_sig("sr_build_prompt", i32, C.c_char_p, i64, C.c_char_p, i64, C.c_char_p, i64, i32, P(i32), i32,
     P(i32), P(i32), i32, P(i32))
_sig("sr_score_result_to_json", i32, C.c_char_p, i32, P(C.c_char_p), i32, P(C.c_char_p), P(f64),
     P(FlopReportC), C.c_char_p, i64, P(i64))
_sig("sr_engine_create", i32, vp, i32, P(vp))
_sig("sr_engine_destroy", None, vp)
_sig("sr_engine_score", i32, vp, P(RequestC), P(ResultC))
_sig("sr_engine_score_batch", i32, vp, P(RequestC), i32, P(ResultC))
_sig("sr_engine_item_hidden", i32, vp, P(RequestC), P(f32))
_sig("sr_engine_set_projection", i32, vp, P(f32), i32, i32)
_sig("sr_engine_reserve", i32, vp, i64)
_sig("sr_engine_score_emb", i32, vp, P(i32), i32, P(f32), i32, i32, P(i64), i32, P(ResultC))
_sig("sr_plan_create_emb", i32, vp, P(i32), i32, P(f32), i32, i32, P(i64), i32, i32, P(vp))
_sig("sr_engine_device", i32, vp)
_sig("sr_engine_stream", vp, vp)
_sig("sr_plan_create", i32, vp, P(RequestC), i32, P(vp))
_sig("sr_plan_create_batch", i32, vp, P(RequestC), i32, i32, P(vp))
_sig("sr_plan_fetch_batch", i32, vp, P(ResultC), i32)
_sig("sr_plan_run", i32, vp)
_sig("sr_plan_sync", i32, vp)
_sig("sr_plan_fetch", i32, vp, P(ResultC))
_sig("sr_plan_kernel_count", i32, vp, P(i32))
_sig("sr_plan_destroy", None, vp)
_sig("sr_plan_profile", i32, vp, i32, P(f32), P(i32))
_sig("sr_plan_shape", i32, vp, P(i64))
class SchedOptionsC(C.Structure):
    _fields_ = [("max_queries", i32), ("max_rows", i64), ("budget_ms", f64),
                ("max_wait_us", i32), ("k", i32), ("borrow", i32), ("sat_rows", i64)]


class SchedStatsC(C.Structure):
    _fields_ = [("submitted", i64), ("completed", i64), ("failed", i64), ("batches", i64),
                ("mean_batch", f64), ("p50_ms", f64), ("p99_ms", f64), ("max_ms", f64),
                ("mean_ms", f64), ("ms_per_row", f64), ("busy_ms", f64),
                ("max_pass_ms", f64), ("max_wait_ms", f64)]


SCHED_EXEC_FN = C.CFUNCTYPE(i32, P(RequestC), i32, P(ResultC), vp)
_sig("sr_sched_create", i32, vp, P(SchedOptionsC), P(vp))
_sig("sr_sched_create_host", i32, P(ModelConfigC), P(SchedOptionsC), SCHED_EXEC_FN, vp, P(vp))
_sig("sr_sched_submit", i32, vp, P(RequestC), P(u64))
_sig("sr_sched_wait", i32, vp, u64, P(ResultC), P(f64), P(i32))
_sig("sr_sched_get_stats", i32, vp, i32, P(SchedStatsC))
_sig("sr_sched_destroy", None, vp)
_sig("sr_nccl_unique_id", i32, P(C.c_uint8))
_sig("sr_comm_create", i32, i32, i32, P(C.c_uint8), i32, P(vp))
ALLGATHER_FN = C.CFUNCTYPE(i32, vp, vp, sz, vp)
_sig("sr_comm_create_host", i32, i32, i32, i32, ALLGATHER_FN, vp, P(vp))
_sig("sr_comm_destroy", None, vp)
_sig("sr_engine_score_sharded", i32, vp, vp, P(RequestC), P(ResultC))
_sig("sr_plan_run_sharded", i32, vp, vp)
_sig("sr_engine_score_b64", i32, vp, P(i32), i32, C.c_char_p, P(i64), i32, P(i64), P(ResultC))
_sig("sr_wire_parse", i32, C.c_char_p, i64, i32, P(vp))
_sig("sr_wire_destroy", None, vp)
_sig("sr_wire_info", i32, vp, P(i32), P(i32), P(i32))
_sig("sr_wire_request_id", C.c_char_p, vp)
_sig("sr_wire_item_id", C.c_char_p, vp, i32)
_sig("sr_engine_score_wire", i32, vp, vp, P(ResultC))
_sig("sr_engine_set_postprocess", i32, vp, P(f64), P(f64), P(f64), i32, P(i32), P(f64), i32)
_sig("sr_engine_final_scores", i32, vp, P(f64), i32, P(i32))
_sig("sr_score_cache_create", i32, i64, P(vp))
_sig("sr_score_cache_destroy", None, vp)
_sig("sr_score_cache_size", i64, vp)
_sig("sr_score_cache_capacity", i64, vp)
_sig("sr_score_cache_get", i32, vp, C.c_char_p, u64, i64, C.c_char_p, P(f64), i32, P(i32))
_sig("sr_score_cache_put", i32, vp, C.c_char_p, u64, i64, C.c_char_p, P(f64), i32)
_sig("sr_canonical_query", i32, C.c_char_p, i32, P(C.c_char_p), P(C.c_char_p), C.c_char_p, i64,
     P(i64))
_sig("sr_query_signature", i32, C.c_char_p, i32, P(C.c_char_p), P(C.c_char_p), P(u64))
_sig("sr_fnv1a64", u64, C.c_char_p, i64)
_sig("sr_engine_score_cached", i32, vp, vp, C.c_char_p, u64, C.c_char_p, P(RequestC), P(ResultC),
     P(i32))
_sig("sr_corpus_create", i32, vp, vp, vp, i64, i32, i32, i32, P(vp))
_sig("sr_corpus_destroy", None, vp)
_sig("sr_corpus_topk", i32, vp, vp, i32, f64, vp, i32, vp, i32, P(i64), P(f64), P(i32))
_sig("sr_corpus_topk_sharded", i32, vp, vp, vp, i32, f64, vp, i32, vp, i32, P(i64), P(f64),
     P(i32))
_sig("sr_corpus_last_candidates", i64, vp)
_sig("sr_corpus_last_scan_ms", f32, vp)
_sig("sr_kernel_gemm", i32, vp, vp, i32, i32, i32, vp, i32, i32, vp)
_sig("sr_kernel_gemm_resid_ln", i32, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp)
_sig("sr_kernel_gemm_ln", i32, vp, vp, i32, i32, i32, vp, i32, i32, vp, vp, i32, vp, i32, vp)
_sig("sr_kernel_attention", i32, vp, P(i32), i32, i32, i32, vp, vp)
_sig("sr_kernel_layernorm", i32, vp, vp, vp, i32, i32, vp)
_sig("sr_debug_attention_trace", i32, vp)
_sig("sr_debug_gemm_trace", i32, vp)
_sig("sr_kernel_topk", i32, vp, vp, i32, i32, P(i64), P(f64), P(i32))

# Every symbol the header declares (tests check the library exports them).
HEADER_SYMBOLS = [
    "sr_last_error", "sr_status_name", "sr_abi_version", "sr_config_validate",
    "sr_config_default_toy", "sr_task_count", "sr_weights_init", "sr_weights_load",
    "sr_weights_save", "sr_weights_from_tensors", "sr_weights_free", "sr_weights_config",
    "sr_weights_version", "sr_weights_tensor_count", "sr_weights_tensor", "sr_flops",
    "sr_multi_item_pair_count", "sr_multi_item_mask", "sr_plan_batches", "sr_request_report",
    "sr_topk_host", "sr_build_prompt", "sr_score_result_to_json",
    "sr_engine_create", "sr_engine_destroy", "sr_engine_score", "sr_engine_score_batch",
    "sr_engine_item_hidden", "sr_engine_reserve", "sr_engine_set_projection", "sr_engine_score_emb",
    "sr_plan_create_emb", "sr_engine_device", "sr_engine_stream", "sr_plan_create",
    "sr_plan_create_batch", "sr_plan_fetch_batch", "sr_plan_run", "sr_plan_sync", "sr_plan_fetch", "sr_plan_kernel_count", "sr_plan_destroy",
    "sr_plan_profile", "sr_plan_shape", "sr_sched_create", "sr_sched_create_host",
    "sr_sched_submit", "sr_sched_wait", "sr_sched_get_stats", "sr_sched_destroy",
    "sr_nccl_unique_id", "sr_comm_create", "sr_comm_create_host", "sr_comm_destroy", "sr_engine_score_sharded",
    "sr_plan_run_sharded", "sr_engine_score_b64", "sr_wire_parse", "sr_wire_destroy",
    "sr_wire_info", "sr_wire_request_id", "sr_wire_item_id", "sr_engine_score_wire", "sr_engine_set_postprocess", "sr_engine_final_scores",
    "sr_score_cache_create", "sr_score_cache_destroy", "sr_score_cache_size",
    "sr_score_cache_capacity", "sr_score_cache_get", "sr_score_cache_put", "sr_canonical_query",
    "sr_query_signature", "sr_fnv1a64", "sr_engine_score_cached", "sr_corpus_create", "sr_corpus_destroy", "sr_corpus_topk",
    "sr_corpus_topk_sharded", "sr_corpus_last_candidates", "sr_corpus_last_scan_ms",
    "sr_kernel_gemm", "sr_kernel_gemm_ln", "sr_kernel_gemm_resid_ln", "sr_kernel_attention", "sr_kernel_layernorm",
    "sr_kernel_topk", "sr_debug_attention_trace", "sr_debug_gemm_trace",
]
