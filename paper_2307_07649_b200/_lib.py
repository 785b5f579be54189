"""ctypes binding of libtgnn_b200.so (the C ABI in include/tgnn_b200.h).

The shared library is the product; this module only marshals arguments and
maps status codes onto exceptions mirroring the reference taxonomy
(ref common.hpp:16-34, tensor.hpp:16). There is no fallback: if the library
is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TGNN_LIB") or os.path.join(HERE, "libtgnn_b200.so")


class TgnnError(RuntimeError):
    code = 8


class ConfigError(TgnnError):
    code = 1


class ParseError(ConfigError):
    code = 2


class NumericError(TgnnError):
    code = 3


class ProtocolError(TgnnError):
    code = 4


class ShapeError(TgnnError):
    code = 5


class CudaError(TgnnError):
    code = 6


class NcclError(TgnnError):
    code = 7


_ERRORS = {1: ConfigError, 2: ParseError, 3: NumericError, 4: ProtocolError, 5: ShapeError,
           6: CudaError, 7: NcclError}

i64 = C.c_int64
i32 = C.c_int32
u64 = C.c_uint64
f64 = C.c_double
vp = C.c_void_p
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)


class ModelConfigC(C.Structure):
    _fields_ = [("d_mem", i64), ("d_time", i64), ("d_static", i64), ("d_attn", i64),
                ("d_hidden", i64), ("d_e", i64), ("n_neighbors", i64), ("num_nodes", i64),
                ("max_t", f64)]


class TrainConfigC(C.Structure):
    _fields_ = [("i", i32), ("j", i32), ("k", i32), ("p", i32), ("q", i32), ("epochs", i32),
                ("local_batch", i64), ("lr_base", f64), ("seed", u64), ("local_batch_ref", i64),
                ("neg_groups", i64)]


class SynthParamsC(C.Structure):
    _fields_ = [("nodes", i64), ("events", i64), ("burst_prob", f64), ("pref_prob", f64),
                ("prefs_per_src", i32), ("src_frac", f64), ("bipartite", i32), ("d_e", i64),
                ("zipf_s", f64), ("seed", u64)]


class RunOptionsC(C.Structure):
    _fields_ = [("model", ModelConfigC), ("train", TrainConfigC), ("train_begin", i64),
                ("train_end", i64), ("rank", i32), ("nranks", i32), ("use_graphs", i32),
                ("val_begin", i64), ("val_end", i64), ("eval_negatives", i32), ("pad0", i32),
                ("eval_batch", i64), ("oplog", i32), ("segment_snapshots", i32)]


_lib = None

# (name, argtypes) -- every entry point declared in include/tgnn_b200.h
SIGNATURES = {
    "tgnn_last_error": [],
    "tgnn_version": [],
    "tgnn_device_count": [C.POINTER(C.c_int)],
    "tgnn_ctx_create": [C.c_int, C.POINTER(vp)],
    "tgnn_ctx_destroy": [vp],
    "tgnn_ctx_synchronize": [vp],
    "tgnn_ctx_stream": [vp, C.POINTER(vp)],
    "tgnn_gen_synthetic": [C.POINTER(SynthParamsC), i64p, i64p, f64p, f32p, i64p],
    "tgnn_graph_create": [vp, i64, i64, i64, i64p, i64p, f64p, f32p, i64, C.POINTER(vp)],
    "tgnn_graph_create_f64": [vp, i64, i64, i64, i64p, i64p, f64p, f64p, i64, C.POINTER(vp)],
    "tgnn_graph_destroy": [vp],
    "tgnn_graph_info": [vp, i64p, i64p, i64p, i64p],
    "tgnn_graph_events": [vp, i64p, i64p, f64p],
    "tgnn_sample_recent_neighbors": [vp, i64p, f64p, i64, i64, i64p, i64p, f64p, i64p],
    "tgnn_sample_negatives": [vp, i64, i64, i64, u64, i64p],
    "tgnn_plan_sub_batch": [vp, i64, i64, i64p, i64, i64p, f64p, i64p, i64p, i64p, f64p, i64p,
                            i64p],
    "tgnn_memstore_create": [vp, i64, i64, C.POINTER(vp)],
    "tgnn_memstore_destroy": [vp],
    "tgnn_memstore_reset": [vp],
    "tgnn_memstore_read": [vp, i64p, i64, f64p, f64p],
    "tgnn_memstore_write": [vp, i64p, i64, f64p, f64p],
    "tgnn_memstore_export": [vp, f64p, f64p, f64p, f64p, f64p, i64p],
    "tgnn_memstore_import": [vp, f64p, f64p, f64p, f64p, f64p, i64p],
    "tgnn_param_count": [C.POINTER(ModelConfigC), i64p],
    "tgnn_init_params": [C.POINTER(ModelConfigC), u64, f64p],
    "tgnn_trainer_create": [vp, vp, C.POINTER(ModelConfigC), i64, u64, C.POINTER(vp)],
    "tgnn_trainer_destroy": [vp],
    "tgnn_trainer_set_params": [vp, f64p],
    "tgnn_trainer_get_params": [vp, f64p],
    "tgnn_trainer_get_grads": [vp, f64p],
    "tgnn_trainer_sub_step": [vp, i64, i64, i64p, f64p, f64p, f64p, f64p],
    "tgnn_trainer_root_writes": [vp, i64p, f64p, f64p, i64p],
    "tgnn_trainer_adam_step": [vp, f64],
    "tgnn_trainer_iterate": [vp, vp, i64, i64, i64, i64, i64, f64, f64p],
    "tgnn_schedule_query": [C.POINTER(TrainConfigC), i64, i64, i32, i64, i64, i64p, i64p],
    "tgnn_comm_unique_id": [C.c_char_p],
    "tgnn_run_create": [vp, vp, C.POINTER(RunOptionsC), C.POINTER(vp)],
    "tgnn_run_comm_init": [vp, C.c_char_p],
    "tgnn_local_hub_create": [i32, C.POINTER(vp)],
    "tgnn_local_hub_destroy": [vp],
    "tgnn_run_local_init": [vp, vp],
    "tgnn_run_destroy": [vp],
    "tgnn_run_info": [vp, i64p, i64p],
    "tgnn_run_barriers": [vp, i64, i64],
    "tgnn_run_losses": [vp, i64, i64, f64p],
    "tgnn_run_params": [vp, f64p],
    "tgnn_run_loss_async": [vp, i64, f64p],
    "tgnn_run_traversed": [vp, i64, i64, i64p],
    "tgnn_run_eval_barriers": [vp, i64p, i64p],
    "tgnn_run_metrics": [vp, i64p, f64p],
    "tgnn_run_oplog": [vp, i64p, i64p],
    "tgnn_run_snapshots": [vp, i64p, i64p, f64p, f64p],
    "tgnn_run_check_replicas": [vp, C.POINTER(C.c_uint64)],
    "tgnn_run_evaluate_mrr": [vp, i64, i64, i64, i32, u64, f64p, i64p],
    "tgnn_evaluator_create": [vp, vp, C.POINTER(ModelConfigC), i64, i32, C.POINTER(vp)],
    "tgnn_evaluator_destroy": [vp],
    "tgnn_evaluate_mrr": [vp, f64p, i64, i64, u64, f64p, i64p],
    "tgnn_replay_batch": [vp, vp, f64p, i64, i64],
    "tgnn_eval_candidates": [vp, i64, i64, u64, i64p],
    "tgnn_checkpoint_save": [C.POINTER(ModelConfigC), f64p, C.c_char_p],
    "tgnn_graph_synthetic": [vp, C.POINTER(SynthParamsC), i32, C.POINTER(vp)],
    "tgnn_graph_load_dataset": [vp, C.c_char_p, i32, C.POINTER(vp)],
    "tgnn_write_dataset": [C.c_char_p, i64, i64, i64, i64p, i64p, f64p, f64p, i64],
    "tgnn_chronological_split": [i64, f64, f64, i64p, i64p],
    "tgnn_graph_edge_feats": [vp, i64, i64, f32p],
    "tgnn_checkpoint_load": [C.POINTER(ModelConfigC), C.c_char_p, f64p],
    "tgnn_run_launches_per_barrier": [vp, i64p],
    "tgnn_run_profile_barrier": [vp, f64p, C.POINTER(C.c_int32), i32],
    "tgnn_run_gemm_profile": [vp, i64, i64p, f64p],
    "tgnn_graph_ingest": [vp, i64, i64, C.POINTER(C.c_int32), C.POINTER(C.c_int32), f64p, f32p],
    "tgnn_pinned_alloc": [i64, C.POINTER(vp)],
    "tgnn_debug_gemm_bench": [i64, i64, i64, i32, i32, f64p, C.POINTER(C.c_uint64), C.POINTER(i32)],
    "tgnn_set_gemm_impl": [C.c_int],
    "tgnn_get_gemm_impl": [C.POINTER(C.c_int)],
    "tgnn_debug_gemm": [C.c_int, i64, i64, i64, f32p, C.c_int, f32p, C.c_int, f32p, C.c_int],
    "tgnn_pinned_free": [vp],
    "tgnn_debug_gru_trace": [C.POINTER(C.c_uint64), i32, C.POINTER(i32)],
}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, argt in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = argt
            fn.restype = C.c_int
        L.tgnn_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        msg = lib().tgnn_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, TgnnError)(msg)
