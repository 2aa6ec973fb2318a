"""ctypes binding of libccwgpu.so (include/ccwgpu.h).

The library is the product: every call below runs on the GPU.  If the shared
object is missing or the device cannot be initialised the calls raise -- there
is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libccwgpu.so")


class SimConfigC(C.Structure):
    _fields_ = [("sg_height", C.c_int32), ("sg_width", C.c_int32),
                ("template_size", C.c_int32), ("overlap", C.c_int32),
                ("dwt_level", C.c_int32), ("candidates", C.c_int32),
                ("n_realizations", C.c_int32), ("scoring", C.c_int32),
                ("facies_mode", C.c_int32), ("min_cut", C.c_int32),
                ("master_seed", C.c_uint64), ("any_support", C.c_int32), ("_pad", C.c_int32)]


class DiagC(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("origin", C.c_int32), ("column_major", C.c_int32),
                ("work_height", C.c_int32), ("work_width", C.c_int32),
                ("placement_count", C.c_int32), ("hard_data_count", C.c_int32),
                ("pre_overwrite_mismatches", C.c_int32), ("_pad", C.c_int32),
                ("wall_seconds", C.c_double)]


class TraceC(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("count", C.c_int32),
                ("top", C.POINTER(C.c_int32)), ("left", C.POINTER(C.c_int32)),
                ("shape", C.POINTER(C.c_int32)), ("ti_row", C.POINTER(C.c_int32)),
                ("ti_col", C.POINTER(C.c_int32)), ("pasted", C.POINTER(C.c_uint8))]


class TimingC(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("ccf_ms", C.c_double), ("select_ms", C.c_double),
                ("ccf_launches", C.c_int64), ("launches", C.c_int64), ("ccf_flop", C.c_double),
                ("ccf_flop_ref", C.c_double), ("waves", C.c_int64), ("jobs", C.c_int64),
                ("rescored", C.c_int64), ("screened_jobs", C.c_int64), ("ccf_variant", C.c_int64),
                ("ccf_mma_flop", C.c_double), ("groups", C.c_int64),
                ("list_overflows", C.c_int64), ("host_prep_ms", C.c_double),
                ("bulk_jobs", C.c_int64), ("shared_groups", C.c_int64), ("d2h_bytes", C.c_int64)]


class Sim3dConfigC(C.Structure):
    _fields_ = [("sg", C.c_int32 * 3), ("template_size", C.c_int32), ("overlap", C.c_int32),
                ("dwt_level", C.c_int32), ("candidates", C.c_int32),
                ("n_realizations", C.c_int32), ("any_support", C.c_int32), ("_pad", C.c_int32),
                ("master_seed", C.c_uint64)]


class Diag3dC(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("corner", C.c_int32), ("order", C.c_int32),
                ("work", C.c_int32 * 3), ("placement_count", C.c_int32),
                ("hard_data_count", C.c_int32), ("pre_overwrite_mismatches", C.c_int32),
                ("wall_seconds", C.c_double)]


P = C.c_void_p
I32P = C.POINTER(C.c_int32)
U8P = C.POINTER(C.c_uint8)
F64P = C.POINTER(C.c_double)
U64P = C.POINTER(C.c_uint64)
INTP = C.POINTER(C.c_int)

# name -> (restype, argtypes); mirrors include/ccwgpu.h one to one.
SIGNATURES = {
    "ccw_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "ccw_ctx_destroy": (None, [P]),
    "ccw_last_error": (C.c_char_p, [P]),
    "ccw_ctx_stream": (P, [P]),
    "ccw_ctx_set_profiling": (C.c_int, [P, C.c_int]),
    "ccw_ctx_last_timing": (C.c_int, [P, C.POINTER(TimingC)]),
    "ccw_ctx_set_ccf_variant": (C.c_int, [P, C.c_int]),
    "ccw_ctx_set_option": (C.c_int, [P, C.c_char_p, C.c_longlong]),
    "ccw_nccl_unique_id": (C.c_int, [U8P]),
    "ccw_ctx_set_position_shards": (C.c_int, [P, C.c_int, C.c_int, U8P, C.c_int]),
    "ccw_measure_fp32_peak": (C.c_int, [P, F64P]),
    "ccw_measure_i8_peak": (C.c_int, [P, F64P]),
    "ccw_measure_int_peak": (C.c_int, [P, C.c_int, F64P]),
    "ccw_measure_ccf_screen": (C.c_int, [P, P, C.c_int, C.c_int, C.c_int, F64P]),
    "ccw_mix64": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "ccw_ti_create": (C.c_int, [P, U8P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(P)]),
    "ccw_ti_create_device": (C.c_int, [P, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(P)]),
    "ccw_ti_destroy": (None, [P]),
    "ccw_ti_apex": (C.c_int, [P, F64P]),
    "ccw_simulate": (C.c_int, [P, P, C.POINTER(SimConfigC), U64P, C.c_int, I32P, C.c_int, U8P,
                               C.POINTER(DiagC), C.POINTER(TraceC)]),
    "ccw_simulate_device": (C.c_int, [P, P, C.POINTER(SimConfigC), U64P, C.c_int, I32P, C.c_int,
                                      P, C.POINTER(DiagC)]),
    "ccw_simulate_device_async": (C.c_int, [P, P, C.POINTER(SimConfigC), U64P, C.c_int, I32P, C.c_int, C.c_void_p]),
    "ccw_ctx_synchronize": (C.c_int, [P]),
    "ccw_simulate_ensemble": (C.c_int, [P, P, C.POINTER(SimConfigC), I32P, C.c_int, U8P,
                                        C.POINTER(DiagC)]),
    "ccw_dwt2_single_f64": (C.c_int, [P, F64P, C.c_int, C.c_int, F64P, F64P, F64P, F64P]),
    "ccw_idwt2_single_f64": (C.c_int, [P, F64P, F64P, F64P, F64P, C.c_int, C.c_int, F64P]),
    "ccw_dwt2_f64": (C.c_int, [P, F64P, C.c_int, C.c_int, C.c_int, F64P, F64P]),
    "ccw_idwt2_f64": (C.c_int, [P, F64P, F64P, C.c_int, C.c_int, C.c_int, F64P]),
    "ccw_score_map_f64": (C.c_int, [P, F64P, F64P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    F64P, C.c_int, F64P]),
    "ccw_top_k_f64": (C.c_int, [P, F64P, C.c_int, C.c_int, C.c_int, I32P, I32P, F64P, INTP]),
    "ccw_select_conditional": (C.c_int, [P, I32P, I32P, C.c_int, I32P, C.c_int, U8P, C.c_int,
                                         C.c_int, C.c_int, INTP, INTP]),
    "ccw_min_cut_stitch": (C.c_int, [P, U8P, U8P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     U8P]),
    "ccw_ti3d_create": (C.c_int, [P, U8P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(P)]),
    "ccw_ti3d_destroy": (None, [P]),
    "ccw_validate_config3d": (C.c_int, [C.POINTER(Sim3dConfigC), I32P, C.c_int, I32P, C.c_int,
                                        C.c_char_p, C.c_size_t]),
    "ccw_simulate3d": (C.c_int, [P, P, C.POINTER(Sim3dConfigC), U64P, C.c_int, I32P, C.c_int, U8P,
                                 C.POINTER(Diag3dC)]),
    "ccw_simulate3d_trace": (C.c_int, [P, P, C.POINTER(Sim3dConfigC), U64P, C.c_int, I32P, C.c_int, U8P,
                                       C.POINTER(Diag3dC), I32P, C.c_int]),
    "ccw_simulate3d_device": (C.c_int, [P, P, C.POINTER(Sim3dConfigC), U64P, C.c_int, I32P, C.c_int,
                                        P, C.POINTER(Diag3dC)]),
    "ccw_simulate3d_ensemble": (C.c_int, [P, P, C.POINTER(Sim3dConfigC), I32P, C.c_int, U8P,
                                          C.POINTER(Diag3dC)]),
    "ccw_variogram": (C.c_int, [P, U8P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, F64P,
                                I32P]),
    "ccw_connectivity": (C.c_int, [P, U8P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   F64P]),
    "ccw_ensemble_average": (C.c_int, [P, U8P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, F64P]),
    "ccw_downsample_majority": (C.c_int, [P, U8P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, U8P]),
    "ccw_pattern_histogram": (C.c_int, [P, U8P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(P)]),
    "ccw_phist_info": (C.c_int, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "ccw_phist_copy": (C.c_int, [P, P, U8P, U64P]),
    "ccw_phist_destroy": (None, [P]),
    "ccw_js_divergence": (C.c_int, [P, P, P, F64P]),
    "ccw_anodi": (C.c_int, [P, U8P, C.c_int, U8P, C.c_int, C.c_int, C.c_int, C.c_int, U8P, C.c_int, C.c_int,
                            C.c_int, C.c_int, C.c_int, F64P, F64P, F64P]),
    "ccw_validate_config": (C.c_int, [C.POINTER(SimConfigC), C.c_int, C.c_int, C.c_int, I32P,
                                      C.c_int, C.c_char_p, C.c_size_t]),
    "ccw_plan_raster_path": (C.c_int, [C.POINTER(SimConfigC), C.c_int, C.c_int, INTP, INTP, I32P,
                                       I32P, I32P, C.c_int, INTP, C.c_char_p, C.c_size_t]),
}

_lib = None


def lib():
    """Load libccwgpu.so (built in-tree by ``__graft_entry__.build()``)."""
    global _lib
    if _lib is None:
        path = os.environ.get("CCW_LIB_VARIANT") or LIB_PATH  # build-variant experiments
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(SIGNATURES)
