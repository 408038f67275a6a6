"""ctypes declarations of include/gsb.h (argument marshalling only).

The product path has no fallback: if libgsb.so is missing or a call fails, an error is
raised.  Nothing here imports or executes oracle/.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libgsb.so")

P = C.c_void_p
i32, i64, u32, u64, f32, sz = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float, C.c_size_t


class gsb_block_view(C.Structure):
    _fields_ = [("dst_gid", P), ("src_gid", P), ("seg_ptr", P), ("e_src_gid", P), ("e_eid", P), ("e_src", P),
                ("num_slots", i32)]


class gsb_sample_args(C.Structure):
    _fields_ = [("seeds", P), ("n_seeds", i64), ("n_seeds_dev", P), ("rng_seed", u64), ("step", u32),
                ("step_dev", P), ("excl_u", P), ("excl_v", P), ("n_excl", i64), ("excl_etype", i32),
                ("excl_rev_etype", i32)]


class gsb_exchange_bufs(C.Structure):
    _fields_ = [("req_send", P), ("req_perm", P), ("send_cnt", P), ("cursor", P), ("req_recv", P), ("cap_recv", i64),
                ("xoff", P), ("srv_meta", P), ("srv_cnt", P), ("srv_seg", P), ("srv_gid", P), ("srv_eid", P),
                ("cap_srv_e", i64), ("srv_wcnt", P), ("resp_cnt", P), ("resp_seg", P), ("resp_gid", P),
                ("resp_eid", P), ("cap_resp_e", i64)]


# gsb_exchange_fn(user, phase, hop, stream, counts)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_int64))

# name -> argtypes (all return gsb_status = int32 unless listed in _RET)
SIGS = {
    "gsb_last_error": [],
    "gsb_version": [],
    "gsb_launch_count": [],
    "gsb_profile_enable": [i32],
    "gsb_profile_dump": [C.c_char_p, sz],
    "gsb_profile_timeline": [C.c_char_p, sz],
    "gsb_graph_create": [i32, P, i32, P, P, C.POINTER(P)],
    "gsb_graph_destroy": [P],
    "gsb_csc_build_bytes": [P, i32, i64, C.POINTER(sz)],
    "gsb_csc_build": [P, i32, P, P, P, i64, P, P, C.POINTER(i64), P, sz, P],
    "gsb_graph_set_csc": [P, i32, P, P, i64, i64],
    "gsb_csc_build_range": [P, i32, P, P, P, i64, i64, i64, P, P, C.POINTER(i64), C.POINTER(i64), P, sz, P],
    "gsb_csc_peers_bytes": [C.POINTER(sz)],
    "gsb_graph_set_csc_peers": [P, P, i32, i32, P, P, P, P, i64, P],
    "gsb_graph_set_features": [P, i32, P, i32, i32],
    "gsb_gather": [P, P, i64, P, P],
    "gsb_blocks_create": [P, i32, P, i64, i64, C.POINTER(P)],
    "gsb_blocks_destroy": [P],
    "gsb_blocks_arena_bytes": [P, C.POINTER(sz)],
    "gsb_blocks_init_arena": [P, P, sz, P],
    "gsb_sample": [P, C.POINTER(gsb_sample_args), P, sz, P],
    "gsb_block_sizes": [P, P, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), P, P, P],
    "gsb_block_view_get": [P, P, i32, C.POINTER(gsb_block_view)],
    "gsb_slot_etype": [P, i32, i32, C.POINTER(i32)],
    "gsb_blocks_poll_error": [P, P, C.POINTER(i32), P],
    "gsb_gather_block_inputs": [P, P, P, P],
    "gsb_blocks_input_rows": [P, C.POINTER(i64)],
    "gsb_blocks_dst_rows": [P, i32, C.POINTER(i64)],
    "gsb_layer_acat_floats": [P, i32, i32, C.POINTER(i64)],
    "gsb_rgcn_layer_fwd": [P, P, i32, P, i32, P, P, i32, i32, P, P, P],
    "gsb_rgcn_layer_fwd_ex": [P, P, i32, P, i32, P, i32, P, P, i32, i32, P, P, P],
    "gsb_rgcn_layer_agg": [P, P, i32, P, i32, P, i32, P, P],
    "gsb_rgcn_layer_gemm": [P, P, i32, P, i32, P, P, i32, i32, P, P],
    "gsb_rgcn_layer_bwd": [P, P, i32, P, P, P, P, i32, i32, i32, P, P, P, P, P],
    "gsb_partition_create": [i32, P, i32, i32, P, C.POINTER(P)],
    "gsb_partition_destroy": [P],
    "gsb_partition_set_shard": [P, i32, P, i32, i32],
    "gsb_bucket_by_owner": [P, P, P, i64, P, P, P, P, P],
    "gsb_shard_gather": [P, P, i64, P, P],
    "gsb_rows_permute": [P, i32, P, P, i64, P, P],
    "gsb_ipc_handle": [P, P, C.POINTER(i64)],
    "gsb_ipc_open": [P, i64, C.POINTER(P)],
    "gsb_ipc_close": [P],
    "gsb_encoder_ws_bytes": [P, P, i32, P],
    "gsb_encoder_fwd": [P, P, P, i32, P, P, sz, P],
    "gsb_encoder_bwd": [P, P, P, P, i32, P, P, sz, P],
    "gsb_graph_set_feature_peers": [P, i32, i32, P, P, i32, i32],
    "gsb_gemm": [i32, P, i64, P, i64, i64, i32, i32, P, i64, P],
    "gsb_gemm_trace": [P, i32],
    "gsb_weight_images_bytes": [i32, i32, i32, C.POINTER(sz)],
    "gsb_weight_images_register": [P, i32, i32, i32, P, sz, P],
    "gsb_weight_images_register_split": [P, i32, i32, i32, P, P],
    "gsb_weight_images_unregister": [P],
    "gsb_weight_images_refresh": [P, i32, P],
    "gsb_blocks_set_exchange": [P, i32, i32, i32, C.POINTER(gsb_exchange_bufs), EXCHANGE_FN, P],
    "gsb_exchange_sizes": [P, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64),
                           C.POINTER(i64)],
    "gsb_nc_loss": [P, i64, i32, P, P, i32, P, P, i64, P, P, P, P, P, P, P],
    "gsb_nc_loss_dw": [P, i64, i32, P, i32, P, P, P, P],
    "gsb_adam_step": [P, P, P, P, i64, f32, f32, f32, f32, i32, P, P],
    "gsb_adam_step_split": [P, P, P, P, i64, f32, f32, f32, f32, i32, P, P, P, i64, i32, i32, i32, P, P, P],
    "gsb_counter_add": [P, i32, P],
    "gsb_spin": [i64, P],
    "gsb_joint_negatives": [i64, i32, i64, i64, u64, u32, P, i64, P, P],
    "gsb_lp_seeds_bytes": [i64, i64, C.POINTER(sz)],
    "gsb_lp_seeds": [P, P, i64, P, i64, P, P, P, P, P, P, sz, P],
    "gsb_lp_score": [P, i64, i32, P, P, P, i64, i32, P, i32, P, P, P, P, P, P],
    "gsb_uniform_negatives": [i64, i32, i64, i64, u64, u32, P, i64, P, P],
    "gsb_construct_features": [P, i32, u32, i64, i64, P, i32, P],
    "gsb_sparse_emb_fwd": [P, P, i32, P, i32, P, P],
    "gsb_blocks_input_rowmap": [P, P, i64, P, P],
    "gsb_nc_predict": [P, i64, i32, P, P, i32, P, P, i64, P, P, P, P],
    "gsb_sparse_adagrad": [P, P, i32, P, P, P, i32, f32, f32, P],
    "gsb_lp_score_ex": [P, i64, i32, P, P, P, i64, i32, i32, i32, P, i32, P, P, P, P, P, P, P, C.c_size_t, P],
    "gsb_lp_score_ws_bytes": [i64, i32, i32, P],
    "gsb_lp_mrr": [P, i64, i64, i32, P, P, P],
    "gsb_sparse_emb_fwd_peers": [P, P, i32, i32, P, P, i32, P, P],
    "gsb_sparse_emb_push": [P, P, i32, i32, P, P, P, P, i32, f32, P],
    "gsb_sparse_adagrad_apply": [P, P, P, P, i64, i32, f32, f32, P],
}
_RET = {"gsb_last_error": C.c_char_p, "gsb_version": i32, "gsb_launch_count": i64}

_lib = None


class GsbError(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise GsbError(f"libgsb.so not built ({SO}); run `python -m paper_2406_06022_b200.build` "
                           "(there is no CPU fallback)")
        L = C.CDLL(SO)
        for name, args in SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _RET.get(name, i32)
        _lib = L
    return _lib


def check(status: int, what: str = ""):
    if status != 0:
        msg = lib().gsb_last_error().decode(errors="replace")
        raise GsbError(f"{what or 'gsb call'} failed (status {status}): {msg}")


def call(name: str, *args):
    """Call gsb_<name>(*args) and raise on a non-OK status."""
    fn = getattr(lib(), name)
    st = fn(*args)
    check(st, name)
    return st
