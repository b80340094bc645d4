"""ctypes binding of libsalient_b200.so (the C-ABI in include/salient_b200.h).

There is no CPU fallback: if the shared library is missing, or CUDA is not
available when a device entry point is called, the call raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

# SAL_LIB: load another build of the same library (A/B of compile-time variants
# by tools/; the product path uses the in-tree build)
LIB_PATH = Path(os.environ.get("SAL_LIB") or
                Path(__file__).resolve().parent / "libsalient_b200.so")

SAL_MAX_HOPS = 8
SAL_RNG_SPLITMIX = 0
SAL_RNG_PHILOX = 1
SAL_MFG_LAST_HOP_EDGES = 1
SAL_MFG_LAST_HOP_FUSED = 2
SAL_SEG_NO_PAD_FILL = 1
SAL_F16 = 1
SAL_F32 = 2
SAL_BF16 = 3

_DTYPE_CODE = {torch.float16: SAL_F16, torch.float32: SAL_F32, torch.bfloat16: SAL_BF16}

vp = ctypes.c_void_p
i64 = ctypes.c_int64
i32 = ctypes.c_int32
u64 = ctypes.c_uint64


class SalGraph(ctypes.Structure):
    _fields_ = [("num_nodes", i64), ("num_edges", i64), ("indptr", vp), ("indices", vp)]


class SalBatchDesc(ctypes.Structure):
    _fields_ = [("batch_id", i64), ("seed_offset", i64), ("n_seeds", i64)]


class SalIdMap(ctypes.Structure):
    _fields_ = [("table", vp), ("table_cap", i64), ("globals", vp), ("globals_cap", i64)]


class SalMfgPlan(ctypes.Structure):
    _fields_ = [("num_hops", i32), ("fanout", i32 * SAL_MAX_HOPS), ("max_seeds", i64),
                ("node_cap", i64 * (SAL_MAX_HOPS + 1)), ("edge_cap", i64 * SAL_MAX_HOPS),
                ("table_cap", i64), ("flags", i32), ("resolve_in_aggregate", i32), ("sample_lanes", i32),
                ("sample_blocks_per_sm", i32), ("aggregate_blocks_per_sm", i32),
                ("reset_in_aggregate", i32)]


class SalMfgLayout(ctypes.Structure):
    _fields_ = [("table", i64), ("globals", i64), ("sizes", i64), ("etot", i64),
                ("dst_indptr", i64 * SAL_MAX_HOPS), ("src_local", i64 * SAL_MAX_HOPS),
                ("src_glob", i64), ("slot", i64), ("rank", i64), ("scan", i64),
                ("scan_bytes", i64), ("total", i64)]


class SalFileHeader(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("version", ctypes.c_uint32),
                ("magic", ctypes.c_uint8 * 4), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("dtype", ctypes.c_int32), ("elem_bytes", ctypes.c_int32),
                ("payload_offset", ctypes.c_int64), ("file_bytes", ctypes.c_int64)]


SAL_EBADMAGIC, SAL_EVERSION, SAL_ETRUNC, SAL_EIO = -10, -11, -12, -13
SAL_FILE_CSR, SAL_FILE_FEAT, SAL_FILE_LABL = 1, 2, 3

P = ctypes.POINTER

# name -> (restype, argtypes); every symbol declared in include/salient_b200.h
SIGNATURES = {
    "sal_version": (ctypes.c_int, []),
    "sal_last_error": (ctypes.c_char_p, []),
    "sal_launch_count": (ctypes.c_longlong, []),
    "sal_hop_key_prefix": (u64, [u64, i64, i64]),
    "sal_mfg_plan_init": (ctypes.c_int, [P(SalMfgPlan), i32, P(i32), i64, i64]),
    "sal_mfg_plan_init_ex": (ctypes.c_int, [P(SalMfgPlan), i32, P(i32), i64, i64, i32]),
    "sal_mfg_layout_init": (ctypes.c_int, [P(SalMfgPlan), P(SalMfgLayout)]),
    "sal_sample_aggregate": (ctypes.c_int, [P(SalGraph), P(SalMfgPlan), P(SalMfgLayout), vp, vp,
                                             u64, i32, vp, i32, i64, i32, vp, i32, i64, i64, vp]),
    "sal_sample_mfg": (ctypes.c_int, [P(SalGraph), P(SalMfgPlan), P(SalMfgLayout), vp, vp, vp,
                                      u64, i32, vp]),
    "sal_scan_ws_bytes": (ctypes.c_size_t, [i64]),
    "sal_idmap_reset": (ctypes.c_int, [P(SalIdMap), vp]),
    "sal_idmap_rehash": (ctypes.c_int, [P(SalIdMap), i64, vp]),
    "sal_idmap_insert": (ctypes.c_int, [P(SalIdMap), vp, i64, vp, vp, vp, vp, vp, vp, vp, vp,
                                        vp]),
    "sal_hop_count": (ctypes.c_int, [P(SalGraph), vp, vp, i64, i32, vp, vp, vp, vp]),
    "sal_hop_sample": (ctypes.c_int, [P(SalGraph), P(SalIdMap), vp, i64, i32, u64, i32, u64, i64,
                                      i32, vp, vp, vp, vp, vp, vp]),
    "sal_hop_sample_tuned": (ctypes.c_int, [P(SalGraph), P(SalIdMap), vp, i64, i32, u64, i32,
                                            u64, i64, i32, vp, vp, vp, vp, vp, i32, i32, vp]),
    "sal_hop_relabel": (ctypes.c_int, [P(SalIdMap), vp, i64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "sal_gather_rows": (ctypes.c_int, [vp, i64, i32, i64, i32, vp, i32, vp, i64, vp, i64, i32,
                                       vp]),
    "sal_gather_labels": (ctypes.c_int, [vp, vp, vp, i64, vp, vp]),
    "sal_segment_mean_fwd": (ctypes.c_int, [vp, vp, vp, i64, vp, i32, i64, i32, vp, i32, i64,
                                            vp]),
    "sal_segment_mean_fwd_ex": (ctypes.c_int, [vp, vp, vp, i64, vp, i32, i64, i32, vp, i32, i64,
                                               i32, vp]),
    "sal_segment_mean_bwd": (ctypes.c_int, [vp, vp, vp, i64, vp, i32, i64, i32, vp, i64, vp]),
    "sal_segment_mean_fwd_global": (ctypes.c_int, [vp, vp, vp, vp, i64, vp, i32, i64, i32, vp,
                                                   i32, i64, vp]),
    "sal_sample_mfg_next": (ctypes.c_int, [P(SalGraph), P(SalMfgPlan), P(SalMfgLayout), vp, vp, vp,
                                           i64, vp, vp, u64, i32, vp]),
    "sal_plan_next": (ctypes.c_int, [vp, i64, vp, vp, vp]),
    "sal_relu_dropout_fwd": (ctypes.c_int, [vp, i64, vp, i64, i64, i32, i32, vp, ctypes.c_float,
                                            u64, vp, vp]),
    "sal_relu_dropout_bwd": (ctypes.c_int, [vp, i64, i32, vp, vp, i64, i32, i64, i32,
                                            ctypes.c_float, vp]),
    "sal_lsm_nll": (ctypes.c_int, [vp, i64, i64, i32, i32, vp, vp, vp, i64, vp]),
    "sal_argmax_correct": (ctypes.c_int, [vp, i64, i64, i32, i32, vp, vp, vp, vp]),
    "sal_transpose_ws_bytes": (ctypes.c_size_t, [i64]),
    "sal_transpose_build": (ctypes.c_int, [vp, vp, vp, i64, i64, i64, vp, vp, vp, vp, i32, vp]),
    "sal_zero_spans": (ctypes.c_int, [vp, vp, i32, vp]),
    "sal_mean_bwd": (ctypes.c_int, [vp, i64, i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp,
                                     i64, vp, vp, ctypes.c_float, vp, i64, i32, vp]),
    "sal_transpose_complex_list": (ctypes.c_int, [i64, P(i64), P(i64)]),
    "sal_mean_bwd_t": (ctypes.c_int, [vp, i64, i32, i32, i64, vp, vp, vp, vp, i64, vp,
                                      ctypes.c_float, vp, i64, i32, vp]),
    "sal_mean_bwd_t_live": (ctypes.c_int, [vp, i64, i32, i32, i64, vp, vp, vp, vp, i64, vp, vp,
                                           ctypes.c_float, vp, i64, i32, vp]),
    "sal_adam_step_tail": (ctypes.c_int, [vp, vp, vp, vp, vp, i64, ctypes.c_float, ctypes.c_float,
                                          ctypes.c_float, ctypes.c_float, vp, i32, vp, vp, vp,
                                          i64, vp, vp, vp]),
    "sal_adam_step": (ctypes.c_int, [vp, vp, vp, vp, vp, i64, ctypes.c_float, ctypes.c_float,
                                     ctypes.c_float, ctypes.c_float, vp, i32, vp]),
    "sal_step_tail": (ctypes.c_int, [vp, vp, vp, i64, vp, vp, vp]),
    "sal_tc_sage_fwd": (ctypes.c_int, [vp, i64, i64, vp, vp, i32, i32, vp, i64, vp, ctypes.c_float,
                                       u64, vp, i32, vp]),
    "sal_tc_gemm_nn": (ctypes.c_int, [vp, i64, i64, vp, i32, vp, i64, i32, vp, i64, i32, vp]),
    "sal_tc_sage_head_ws_bytes": (ctypes.c_size_t, [i64, i32, i32]),
    "sal_tc_sage_head": (ctypes.c_int, [vp, i64, i64, vp, i32, vp, i64, i32, i32, vp, i64, vp,
                                        vp, i64, vp, i64, vp, i64, vp, ctypes.c_size_t, vp]),
    "sal_tc_sage_logits_argmax": (ctypes.c_int, [vp, i64, i64, vp, i32, vp, i64, i32, i32, vp,
                                                 i64, vp, vp, ctypes.c_size_t, vp]),
    "sal_tc_sage_wgrad": (ctypes.c_int, [vp, i64, vp, i64, i64, vp, i32, i32, vp, i64, i32, vp]),
    "sal_gen_degrees": (ctypes.c_int, [i64, u64, ctypes.c_double, ctypes.c_double, vp, vp]),
    "sal_gen_owner": (ctypes.c_int, [vp, i64, vp, vp]),
    "sal_gen_pairing": (ctypes.c_int, [vp, i64, u64, vp, vp]),
    "sal_gen_features_uniform": (ctypes.c_int, [i64, i32, i64, u64, vp, vp]),
    "sal_gen_labels_uniform": (ctypes.c_int, [i64, i32, u64, vp, vp]),
    "sal_file_header_read": (ctypes.c_int, [ctypes.c_char_p, i32, P(SalFileHeader)]),
    "sal_load_csr": (ctypes.c_int, [ctypes.c_char_p, P(SalFileHeader), vp, vp, vp, i64, i32, vp]),
    "sal_load_features": (ctypes.c_int, [ctypes.c_char_p, P(SalFileHeader), vp, i64, vp, vp, i64,
                                         i32, vp]),
    "sal_load_labels": (ctypes.c_int, [ctypes.c_char_p, P(SalFileHeader), vp, vp, vp, i64, i32,
                                       vp]),
    "sal_validate_csr": (ctypes.c_int, [vp, vp, i64, i64, vp, vp]),
    "sal_validate_labels": (ctypes.c_int, [vp, i64, i64, vp, vp]),
}


class SalError(RuntimeError):
    pass


_LIB = None


def lib():
    """Load the library (raises if it has not been built)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise SalError(f"{LIB_PATH.name} is not built; run `python -c 'import "
                           f"__graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().sal_last_error().decode(errors="replace")
        raise SalError(f"{what or 'salient_b200'} failed ({rc}): {msg}")


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise SalError("salient_b200 device path called without a CUDA device "
                       "(there is no CPU fallback)")


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _DTYPE_CODE[dt]
    except KeyError:
        raise ValueError(f"unsupported dtype {dt}") from None
