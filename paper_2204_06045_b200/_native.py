"""Loader for the in-tree native library ``libqtng.so`` (C ABI: include/qtng.h).

There is no fallback: if the library is missing or fails to load, importing
the package raises.  Build it with ``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_2204_06045_b200/csrc``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.environ.get("QTNG_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libqtng.so")  # override: kernel tuning runs

i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


class Record(C.Structure):
    """qtng_record == qtnsim::TimingRecord (engine.hpp:71-80)."""

    _fields_ = [("edge_u", C.c_int32), ("edge_v", C.c_int32), ("bucket_seq", C.c_int32),
                ("width", C.c_int32), ("elapsed_s", C.c_double), ("ops", C.c_uint64),
                ("flops_est", C.c_double)]


class PlanInfo(C.Structure):
    _fields_ = [("n_lightcones", C.c_int32), ("n_levels", C.c_int32),
                ("n_buckets", C.c_uint64), ("n_device_ops", C.c_uint64),
                ("max_width", C.c_int32), ("max_result_rank", C.c_int32),
                ("alg_bytes", C.c_double), ("sum_ops", C.c_double),
                ("arena_bytes", C.c_uint64), ("desc_bytes", C.c_uint64),
                ("kernels_per_run", C.c_int32), ("n_segments", C.c_uint64),
                ("n_fused_ops", C.c_uint64), ("dev_bytes", C.c_double),
                ("fp64_ops", C.c_double), ("seg_fp64_ops", C.c_double),
                ("single_alg_bytes", C.c_double)]


class EnergyReport(C.Structure):
    """qtng_energy_report: ContractionReport's aggregate fields (engine.hpp:82-88)."""

    _fields_ = [("records", C.c_void_p), ("rec_cap", C.c_int64), ("n_records", C.c_int64),
                ("peak_tensor_bytes", C.c_uint64), ("merges_applied", C.c_int32),
                ("merges_skipped", C.c_int32), ("device_ms", C.c_float)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"native library {LIB_PATH} is missing; build it first "
                          "(make -C paper_2204_06045_b200/csrc)")
    lib = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    pvp = C.POINTER(C.c_void_p)
    lib.qtng_last_error.restype = C.c_char_p
    lib.qtng_version.restype = C.c_char_p
    lib.qtng_create.argtypes = [C.c_int, C.c_uint64, pvp]
    lib.qtng_destroy.argtypes = [vp]
    lib.qtng_destroy.restype = None
    lib.qtng_random_regular.argtypes = [C.c_int, C.c_int, C.c_uint64, i32p, C.c_int,
                                        C.POINTER(C.c_int)]
    lib.qtng_edge_schedule.argtypes = [C.c_int, C.c_int, i32p, C.c_int, f64p, f64p, C.c_int,
                                       C.c_int, i32p, C.c_int64, f64p, C.c_int64,
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int), C.c_void_p]
    lib.qtng_simulate_widths.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int, C.c_int,
                                         i32p, C.c_int, C.POINTER(C.c_int)]
    lib.qtng_edge_costs.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int, f64p]
    lib.qtng_edge_work.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int, f64p]
    lib.qtng_validate_energy.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int, C.c_int]
    lib.qtng_plan_dump.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_void_p, i32p, C.c_int64, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int)]
    lib.qtng_contract_bucket.argtypes = [vp, C.c_int, i32p, i32p, f64p, C.c_int, i32p,
                                         C.POINTER(C.c_int), i32p, f64p, C.c_int64]
    lib.qtng_contract_schedule.argtypes = [vp, C.c_int, i32p, C.c_int64, f64p, C.c_int, f64p,
                                           C.POINTER(Record), C.c_int, C.POINTER(C.c_int),
                                           C.POINTER(C.c_uint64)]
    lib.qtng_energy.argtypes = [vp, C.c_int, C.c_int, i32p, C.c_int, f64p, f64p, C.c_int,
                                C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_double),
                                f64p, C.POINTER(EnergyReport)]
    lib.qtng_energy_multi.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, i32p,
                                      C.c_int, f64p, f64p, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_double), f64p, f32p]
    lib.qtng_shard_edges.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int, C.c_int, i32p]
    lib.qtng_plan_create.argtypes = [vp, C.c_int, C.c_int, i32p, C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.c_int, C.c_void_p, pvp]
    lib.qtng_plan_terms.argtypes = [vp, f64p]
    lib.qtng_merge_schedule.argtypes = [C.c_int, i32p, C.c_int64, C.c_void_p, C.c_int64,
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int), C.c_void_p]
    lib.qtng_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.qtng_plan_create_schedule.argtypes = [vp, C.c_int, i32p, C.c_int64, f64p, C.c_int, pvp]
    lib.qtng_plan_execute.argtypes = [vp, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.POINTER(C.c_float)]
    lib.qtng_plan_profile.argtypes = [vp, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.POINTER(C.c_float)]
    lib.qtng_plan_run_device.argtypes = [vp, C.c_int, C.POINTER(C.c_float)]
    lib.qtng_plan_info_get.argtypes = [vp, C.POINTER(PlanInfo)]
    lib.qtng_kernel_launches.argtypes = []
    lib.qtng_kernel_launches.restype = C.c_uint64
    lib.qtng_set_precision.argtypes = [vp, C.c_int]
    lib.qtng_statevector_energy.argtypes = [vp, C.c_int, C.c_int, i32p, C.c_int, f64p, f64p,
                                            C.c_int, C.POINTER(C.c_double), C.c_void_p]
    lib.qtng_plan_segments.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int, C.c_int, i32p,
                                       C.c_int64, C.POINTER(C.c_int64)]
    lib.qtng_plan_stats.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(PlanInfo)]
    lib.qtng_plan_records.argtypes = [vp, C.POINTER(Record), C.c_int64, C.POINTER(C.c_int64)]
    lib.qtng_plan_level_ms.argtypes = [vp, f32p, C.c_int]
    lib.qtng_plan_kernel_ms.argtypes = [vp, f32p, C.c_void_p, C.c_int]
    lib.qtng_plan_destroy.argtypes = [vp]
    lib.qtng_plan_destroy.restype = None
    lib.qtng_plan_time_level.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_int),
                                         C.POINTER(C.c_double), C.POINTER(C.c_float)]
    return lib


lib = _load()

# Every symbol include/qtng.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "qtng_create", "qtng_destroy", "qtng_last_error", "qtng_version", "qtng_random_regular",
    "qtng_edge_schedule", "qtng_simulate_widths", "qtng_edge_costs", "qtng_edge_work", "qtng_validate_energy", "qtng_plan_dump", "qtng_contract_bucket",
    "qtng_contract_schedule", "qtng_energy", "qtng_energy_multi", "qtng_shard_edges", "qtng_plan_terms", "qtng_merge_schedule", "qtng_fp64_peak", "qtng_plan_create", "qtng_plan_create_schedule", "qtng_plan_execute", "qtng_plan_profile",
    "qtng_plan_run_device", "qtng_plan_info_get", "qtng_plan_stats", "qtng_kernel_launches", "qtng_set_precision", "qtng_statevector_energy", "qtng_plan_segments", "qtng_plan_records", "qtng_plan_level_ms", "qtng_plan_kernel_ms",
    "qtng_plan_destroy", "qtng_plan_time_level",
]
