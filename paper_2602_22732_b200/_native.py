"""ctypes binding of libgr4ad.so (include/gr4ad.h).

The product path has no CPU fallback: importing this module raises if the
sm_100a library is missing, and every entry point raises on a non-OK status
(``ValueError`` for the reference's argument errors, ``RuntimeError`` for
CUDA failures) -- mirroring how ``beam_search`` raises (beam.py:125-132).
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GR4AD_LIB: an instrumented build (e.g. GR_FUSED_TIMING, profiles/fused_phases.py)
LIB_PATH = os.environ.get("GR4AD_LIB") or os.path.join(_HERE, "libgr4ad.so")

MAX_LEVELS = 8
MAX_LAYERS = 32
MAX_BEAM = 8192

OK, ERR_VALUE, ERR_UNSUPPORTED, ERR_WORKSPACE, ERR_CUDA, ERR_RANGE = range(6)


class RangeError(RuntimeError):
    """An operand left the fp16 split range of the tensor-core paths
    (GR4AD_ERR_RANGE): |weight| >= 32 or |context X| >= 256.  The decode
    API retries such batches on the CUDA-core path when ``path="auto"``."""

KERNEL_CLASSES = ("gemm", "attn_gemm", "topk_select", "softmax", "layernorm", "self_attn",
                  "row_lse", "small", "collect", "fused_decode")

EXPORTS = (
    "gr4ad_abi_version", "gr4ad_last_error", "gr4ad_status_string",
    "gr4ad_take_launch_count", "gr4ad_profile_begin", "gr4ad_profile_end",
    "gr4ad_workspace_bytes", "gr4ad_beam_search", "gr4ad_prepare",
    "gr4ad_beam_search_run", "gr4ad_context_process", "gr4ad_encoder_kv",
    "gr4ad_topk_precut", "gr4ad_topk_workspace_bytes", "gr4ad_project_topk",
    "gr4ad_project_topk_workspace_bytes", "gr4ad_gemm", "gr4ad_score_sequences",
    "gr4ad_score_workspace_bytes", "gr4ad_range_status", "gr4ad_prepare_weights",
    "gr4ad_gemm_presplit", "gr4ad_range_flag_offset", "gr4ad_encode_trunk",
    "gr4ad_level_step", "gr4ad_collect", "gr4ad_topk_precut_f64", "gr4ad_resolve_items",
    "gr4ad_derived_layout",
)

_P = C.c_void_p


class Dims(C.Structure):
    _fields_ = [("feat_dim", C.c_int), ("d", C.c_int), ("d_ff", C.c_int),
                ("n_layers", C.c_int), ("trunk_depth", C.c_int), ("n_levels", C.c_int),
                ("n_value_buckets", C.c_int), ("vocab", C.c_int * MAX_LEVELS)]


class Layer(C.Structure):
    _fields_ = [(n, _P) for n in (
        "ln1_g", "ln1_b", "cross_Wq", "cross_Wo", "ln2_g", "ln2_b", "self_Wqkv",
        "self_Wo", "ln3_g", "ln3_b", "ffn_W1", "ffn_b1", "ffn_W2", "ffn_b2")]


class Weights(C.Structure):
    _fields_ = [("ctx_W", _P), ("ctx_b", _P), ("pos", _P), ("bos", _P),
                ("emb", _P * MAX_LEVELS), ("head", _P * MAX_LEVELS),
                ("head_value", _P), ("fuse_Wg", _P), ("fuse_Wf", _P),
                ("cross_kv_W", _P), ("layer", Layer * MAX_LAYERS)]


class Batch(C.Structure):
    _fields_ = [("n_requests", C.c_int), ("ctx_len", C.POINTER(C.c_int)),
                ("widths", C.POINTER(C.c_int)), ("trunk_depth", C.c_int),
                ("value_rerank", C.c_int), ("value_reps", _P),
                ("valid_prefix", _P * MAX_LEVELS),
                ("valid_prefix_count", C.POINTER(C.c_int)), ("decode_path", C.c_int),
                ("weights_prepared", C.c_int), ("derived", _P), ("derived_bytes", C.c_size_t)]

PATH_AUTO, PATH_LAYERED, PATH_FUSED = 0, 1, 2


class Results(C.Structure):
    _fields_ = [("max_out", C.c_int), ("count", _P), ("tokens", _P), ("score", _P)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name in EXPORTS:
        getattr(lib, name)  # AttributeError if an export is missing
    lib.gr4ad_last_error.restype = C.c_char_p
    lib.gr4ad_status_string.restype = C.c_char_p
    lib.gr4ad_status_string.argtypes = [C.c_int]
    lib.gr4ad_take_launch_count.restype = C.c_longlong
    lib.gr4ad_profile_end.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_longlong), C.c_int]
    lib.gr4ad_workspace_bytes.argtypes = [C.POINTER(Dims), C.POINTER(Batch),
                                          C.POINTER(C.c_size_t), C.POINTER(C.c_int)]
    run_args = [C.POINTER(Dims), C.POINTER(Weights), C.POINTER(Batch), _P, _P,
                C.POINTER(Results), _P, C.c_size_t, _P]
    lib.gr4ad_beam_search.argtypes = run_args
    lib.gr4ad_beam_search_run.argtypes = run_args
    lib.gr4ad_prepare.argtypes = [C.POINTER(Dims), C.POINTER(Batch), _P, C.c_size_t, _P]
    lib.gr4ad_range_status.argtypes = [C.POINTER(Dims), C.POINTER(Batch), _P, _P]
    lib.gr4ad_prepare_weights.argtypes = [C.POINTER(Dims), C.POINTER(Weights), C.POINTER(Batch),
                                          _P, C.c_size_t, _P]
    lib.gr4ad_context_process.argtypes = [C.POINTER(Dims), C.POINTER(Weights), _P, C.c_int,
                                          _P, _P]
    lib.gr4ad_encoder_kv.argtypes = [C.POINTER(Dims), C.POINTER(Weights), _P, C.c_int,
                                     C.c_int, C.c_int, _P, _P]
    lib.gr4ad_topk_precut.argtypes = [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P,
                                      _P, _P, _P, C.c_size_t, _P]
    lib.gr4ad_topk_workspace_bytes.restype = C.c_size_t
    lib.gr4ad_topk_workspace_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
    lib.gr4ad_project_topk.argtypes = [_P, _P, C.c_int, _P, C.c_int, C.c_int, C.c_int,
                                       C.c_int, _P, _P, _P, _P, _P, C.c_size_t, _P]
    lib.gr4ad_project_topk_workspace_bytes.restype = C.c_size_t
    lib.gr4ad_project_topk_workspace_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
    lib.gr4ad_gemm.argtypes = [_P, C.c_longlong, _P, C.c_longlong, _P, C.c_longlong, C.c_int,
                               C.c_int, C.c_int, C.c_int, _P]
    lib.gr4ad_gemm_presplit.argtypes = [_P, _P, C.c_longlong, _P, _P, C.c_longlong, _P,
                                        C.c_longlong, C.c_int, C.c_int, C.c_int, C.c_float, _P]
    lib.gr4ad_score_sequences.argtypes = [C.POINTER(Dims), C.POINTER(Weights), C.POINTER(Batch),
                                          _P, _P, C.c_int, C.POINTER(C.c_int), _P, _P, _P, _P,
                                          _P, C.c_size_t, _P]
    lib.gr4ad_score_workspace_bytes.argtypes = [C.POINTER(Dims), C.POINTER(Batch), C.c_int,
                                                C.POINTER(C.c_size_t)]
    lib.gr4ad_range_flag_offset.argtypes = [C.POINTER(Dims), C.POINTER(Batch),
                                            C.POINTER(C.c_size_t)]
    lib.gr4ad_encode_trunk.argtypes = [C.POINTER(Dims), C.POINTER(Weights), C.POINTER(Batch),
                                       _P, _P, _P, C.c_size_t, _P]
    lib.gr4ad_level_step.argtypes = [C.POINTER(Dims), C.POINTER(Weights), C.POINTER(Batch),
                                     C.c_int, _P, C.c_size_t, _P]
    lib.gr4ad_collect.argtypes = [C.POINTER(Dims), C.POINTER(Batch), C.POINTER(Results), _P,
                                  C.c_size_t, _P]
    lib.gr4ad_topk_precut_f64.argtypes = [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P,
                                          _P, _P, _P]
    lib.gr4ad_resolve_items.argtypes = [_P, _P, C.c_int, C.POINTER(Dims), C.POINTER(Results),
                                        C.c_int, _P, _P]
    lib.gr4ad_derived_layout.argtypes = [C.POINTER(Dims), C.POINTER(Batch),
                                         C.POINTER(C.c_size_t), C.POINTER(C.c_ulonglong)]
    if lib.gr4ad_abi_version() != 2:
        raise ImportError("libgr4ad ABI version mismatch")
    return lib


lib = _load()


def check(status):
    if status == OK:
        return
    msg = lib.gr4ad_last_error().decode(errors="replace")
    if status == ERR_VALUE:
        raise ValueError(msg)
    kind = lib.gr4ad_status_string(status).decode()
    if status == ERR_RANGE:
        raise RangeError(f"libgr4ad: {kind}: {msg}")
    raise RuntimeError(f"libgr4ad: {kind}: {msg}")
