"""ctypes declarations for libmggcn.so (include/mggcn.h). Loading fails loudly when the library is missing:
there is no CPU or PyTorch fallback for the device path."""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# MGGCN_RACECHECK=1 loads the racecheck variant of the same sources (build.py --racecheck; sanitizer runs only)
LIB_PATH = os.path.join(PKG, "libmggcn_rc.so" if os.environ.get("MGGCN_RACECHECK") == "1" else "libmggcn.so")

c_i64p = C.POINTER(C.c_int64)


class mg_csr(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("values", C.c_void_p)]


class mg_config(C.Structure):
    _fields_ = [("layer_dims", C.c_void_p), ("n_dims", C.c_int32), ("lr", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("epsilon", C.c_double), ("epochs", C.c_int32), ("seed", C.c_uint64),
                ("permute", C.c_uint8), ("overlap", C.c_uint8), ("skip_first_backward_spmm", C.c_uint8),
                ("order_swap", C.c_uint8), ("gemm_mode", C.c_int32), ("spmm_mode", C.c_int32),
                ("aggregate_input", C.c_int32), ("bias", C.c_int32), ("dropout", C.c_double)]


class mg_timeline_event(C.Structure):
    _fields_ = [("worker", C.c_int32), ("lane", C.c_int32), ("stage", C.c_int32), ("n_deps", C.c_int32),
                ("kind", C.c_char * 16), ("op", C.c_char * 16), ("t_start_us", C.c_double),
                ("t_end_us", C.c_double), ("task", C.c_uint64), ("deps", C.POINTER(C.c_uint64))]


# (name, restype, argtypes) for every symbol declared in include/mggcn.h
SIGNATURES = [
    ("mg_config_defaults", None, [C.c_void_p]),
    ("mg_config_validate", C.c_int, [C.c_void_p]),
    ("mg_last_error", C.c_char_p, []),
    ("mg_abi_version", C.c_int32, []),
    ("mg_set_tuning", C.c_int, [C.c_char_p, C.c_int64]),
    ("mg_dataset_synth", C.c_int, [C.c_int64, C.c_double, C.c_double, C.c_uint64, C.c_int64, C.c_int32, C.c_void_p]),
    ("mg_dataset_from_arrays", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_dataset_view", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_dataset_num_classes", C.c_int32, [C.c_void_p]),
    ("mg_dataset_validate", C.c_int, [C.c_void_p]),
    ("mg_dataset_free", None, [C.c_void_p]),
    ("mg_dataset_masks", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_dataset_load", C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_void_p]),
    ("mg_graph_load", C.c_int, [C.c_char_p, C.c_int32, C.c_void_p]),
    ("mg_graph_view", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mg_graph_free", None, [C.c_void_p]),
    ("mg_dense_load", C.c_int, [C.c_char_p, C.c_void_p]),
    ("mg_dense_read", C.c_int, [C.c_char_p, C.c_void_p]),
    ("mg_dense_view", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_dense_free", None, [C.c_void_p]),
    ("mg_dense_write", C.c_int, [C.c_char_p, C.c_int64, C.c_int64, C.c_void_p]),
    ("mg_graph_from_coo", C.c_int, [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_graph_add_self_loops", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mg_checkpoint_write", C.c_int, [C.c_char_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_checkpoint_read", C.c_int, [C.c_char_p, C.c_void_p]),
    ("mg_checkpoint_count", C.c_int32, [C.c_void_p]),
    ("mg_checkpoint_view", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_checkpoint_free", None, [C.c_void_p]),
    ("mg_config_to_json", C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.c_int64, C.c_void_p]),
    ("mg_breakdown_to_json", C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.c_int64, C.c_void_p]),
    ("mg_breakdown_text", C.c_int, [C.c_void_p, C.c_char_p, C.c_int64, C.c_void_p]),
    ("mg_group_abort", C.c_int, [C.c_void_p]),
    ("mg_labels_load", C.c_int, [C.c_char_p, C.c_void_p, C.c_int64, C.c_void_p]),
    ("mg_masks_load", C.c_int, [C.c_char_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_prepare", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    ("mg_prepare_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    ("mg_partition_info", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_partition_tile_info", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                         C.c_void_p]),
    ("mg_partition_tile_export", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                           C.c_void_p]),
    ("mg_partition_rows_export", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_partition_rows_info", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_partition_free", None, [C.c_void_p]),
    ("mg_synth_rank_open", C.c_int, [C.c_int64, C.c_double, C.c_double, C.c_uint64, C.c_int64, C.c_int32,
                                     C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    ("mg_synth_rank_info", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_synth_rank_degrees", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mg_synth_rank_block_degrees", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    ("mg_synth_rank_finish", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_synth_rank_free", None, [C.c_void_p]),
    ("mg_device_count", C.c_int32, []),
    ("mg_nccl_unique_id", C.c_int, [C.c_void_p]),
    ("mg_group_create", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_int32, C.c_void_p]),
    ("mg_group_init_params", C.c_int, [C.c_void_p]),
    ("mg_group_train_step", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_group_compute_gradients", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_group_loss_only", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mg_group_forward", C.c_int, [C.c_void_p]),
    ("mg_group_train_step_async", C.c_int, [C.c_void_p, C.c_int32]),
    ("mg_group_sync", C.c_int, [C.c_void_p]),
    ("mg_group_last_stats", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_group_read", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64]),
    ("mg_group_write", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64]),
    ("mg_group_w_hash", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    ("mg_group_rows", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    ("mg_group_buffer_audit", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_group_last_profile", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_group_graph_steps", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("mg_group_backward", C.c_int, [C.c_void_p]),
    ("mg_group_destroy", None, [C.c_void_p]),
    ("mg_group_set_timeline", C.c_int, [C.c_void_p, C.c_int32]),
    ("mg_group_timeline", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    ("mg_timeline_export", C.c_int, [C.c_char_p, C.c_void_p, C.c_int64]),
    ("mg_timeline_audit", C.c_int, [C.c_void_p, C.c_int64]),
    ("mg_timeline_audit_staged", C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32]),
    ("mg_timeline_breakdown", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    ("mg_group_bench_spmm", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    ("mg_dev_spmm", C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                              C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    ("mg_dev_gemm", C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                              C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p]),
    ("mg_dev_softmax_xent", C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                      C.c_void_p, C.c_void_p]),
    ("mg_dev_adam", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_double,
                              C.c_double, C.c_double, C.c_int32, C.c_void_p]),
]

_lib = None


def lib():
    """The loaded libmggcn.so. Raises if it was not built — the device path has no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2110_08688_b200.build` "
                               "(the MG-GCN device path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
