"""ctypes binding of libatkg.so (include/atkg.h).

This is the same binding a maintainer would add on the reference side for a
Python caller.  There is deliberately no fallback: if the
CUDA library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ATKG_LIB") or os.path.join(_HERE, "libatkg.so")  # override: experiments only

ATKG_OK, ATKG_EINVAL, ATKG_ENAN, ATKG_EINFEASIBLE, ATKG_ECUDA, ATKG_EUNSUPPORTED, ATKG_EFORMAT = range(7)
ATKG_F32, ATKG_BF16 = 0, 1
OP_STAGE1, OP_APPROX, OP_SELECT, OP_EXACT, OP_SUMMARY, OP_MERGE = range(6)
FLAG_NAN = 1


class NoFeasibleConfigError(RuntimeError):
    """atk::NoFeasibleConfigError (planner.hpp:14-16)."""


class DatasetFormatError(RuntimeError):
    """atk::DatasetFormatError (dataset.hpp:14-16)."""


class Params(C.Structure):
    _fields_ = [("n", C.c_uint64), ("num_buckets", C.c_uint64), ("local_k", C.c_uint32),
                ("global_k", C.c_uint32), ("lane_multiple", C.c_uint32)]


class PlanRequestC(C.Structure):
    _fields_ = [("n", C.c_uint64), ("k", C.c_uint64), ("recall_target", C.c_double),
                ("allowed_local_k", C.POINTER(C.c_uint32)), ("num_allowed_local_k", C.c_uint32),
                ("lane_multiple", C.c_uint32), ("seed", C.c_uint64)]


class PlanResultC(C.Structure):
    _fields_ = [("local_k", C.c_uint32), ("num_buckets", C.c_uint64), ("num_elements", C.c_uint64),
                ("recall", C.c_double), ("recall_method", C.c_int),
                ("recall_std_error", C.c_double), ("recall_trials", C.c_uint64),
                ("high_target_warning", C.c_int)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2506_04165_b200/build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER(Params)
    vp, u64, u32, i32, f64p = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(C.c_double)
    sz = C.POINTER(C.c_size_t)
    sigs = {
        "atkg_last_error": ([], C.c_char_p),
        "atkg_version": ([], C.c_char_p),
        "atkg_set_device": ([i32], i32),
        "atkg_set_option": ([C.c_char_p, u64], i32),
        "atkg_get_option": ([C.c_char_p, u64], u64),
        "atkg_validate": ([P], i32),
        "atkg_validate_analysis": ([P], i32),
        "atkg_workspace_size": ([i32, i32, u64, P, sz], i32),
        "atkg_stage1": ([i32, vp, u64, P, vp, vp, vp, C.c_size_t, vp, vp], i32),
        "atkg_select_candidates": ([vp, vp, u64, u64, u64, u32, u64, vp, vp, vp, C.c_size_t, vp, vp], i32),
        "atkg_approx_top_k": ([i32, vp, u64, P, vp, vp, vp, C.c_size_t, vp, vp], i32),
        "atkg_exact_top_k": ([i32, vp, u64, u64, u32, vp, vp, vp, C.c_size_t, vp, vp], i32),
        "atkg_stage1_summary": ([i32, vp, u64, u64, P, vp, vp, C.c_size_t, vp, vp], i32),
        "atkg_summary_merge_top_k": ([vp, u32, P, vp, vp, vp, vp, vp, C.c_size_t, vp, vp], i32),
        "atkg_check_status": ([vp, vp], i32),
        "atkg_slice_payload_words": ([P, u32, sz], i32),
        "atkg_slice_payload_workspace": ([i32, u64, P, u32, sz], i32),
        "atkg_slice_payload": ([i32, vp, u64, u64, P, u32, vp, vp, C.c_size_t, vp, vp], i32),
        "atkg_payload_merge_top_k": ([vp, u32, P, vp, vp, vp, vp, vp], i32),
        "atkg_sharded_workspace_size": ([i32, u64, P, u32, sz], i32),
        "atkg_sharded_approx_top_k": ([i32, vp, u64, u64, P, vp, u32, vp, vp, vp, C.c_size_t, vp, vp], i32),
        "atkg_nccl_unique_id": ([C.c_char_p], i32),
        "atkg_nccl_comm_init": ([C.POINTER(vp), i32, C.c_char_p, i32], i32),
        "atkg_nccl_comm_destroy": ([vp], i32),
        "atkg_accumulator_create": ([P, C.POINTER(vp)], i32),
        "atkg_accumulator_consume": ([vp, i32, vp, u64, vp], i32),
        "atkg_accumulator_consumed": ([vp], u64),
        "atkg_accumulator_candidates": ([vp, vp, vp, vp], i32),
        "atkg_accumulator_destroy": ([vp], None),
        "atkg_fused_gemm_top_k": ([vp, vp, u64, u64, P, vp, vp, vp, vp, C.c_size_t, vp, vp], i32),
        "atkg_fused_workspace_size": ([u64, u64, P, sz], i32),
        "atkg_gemm_bf16": ([vp, vp, u64, u64, u64, vp, vp], i32),
        "atkg_stage1_host": ([vp, u64, P, vp, vp], i32),
        "atkg_select_candidates_host": ([vp, vp, u64, u32, u64, vp, vp], i32),
        "atkg_approx_top_k_host": ([vp, u64, P, vp, vp], i32),
        "atkg_exact_top_k_host": ([vp, u64, u32, vp, vp], i32),
        "atkg_measure_recall": ([vp, u64, vp, u64, f64p], i32),
        "atkg_exact_expected_recall": ([P, f64p], i32),
        "atkg_mc_expected_recall": ([P, u64, u64, f64p, f64p], i32),
        "atkg_mc_expected_recall_adaptive": ([P, u64, f64p, f64p, C.POINTER(C.c_uint64)], i32),
        "atkg_legal_bucket_counts": ([u64, u64, vp, u64], u64),
        "atkg_select_parameters": ([C.POINTER(PlanRequestC), C.POINTER(PlanResultC)], i32),
        "atkg_approx_top_k_at_recall_host": ([vp, u64, C.POINTER(PlanRequestC), C.POINTER(PlanResultC), vp, vp], i32),
        "atkg_approx_at_recall_workspace_size": ([i32, u64, C.POINTER(PlanRequestC), sz], i32),
        "atkg_approx_top_k_at_recall": ([i32, vp, u64, C.POINTER(PlanRequestC), C.POINTER(PlanResultC), vp, vp, vp,
                                         C.c_size_t, vp, vp], i32),
        "atkg_accumulator_consume_host": ([vp, vp, u64], i32),
        "atkg_accumulator_candidates_host": ([vp, vp, vp], i32),
        "atkg_dataset_read_header": ([C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)], i32),
        "atkg_dataset_read_file": ([C.c_char_p, vp, u64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)], i32),
        "atkg_dataset_write_file": ([C.c_char_p, vp, u64, u64], i32),
        "atkg_dataset_read_file_device": ([C.c_char_p, vp, u64, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64), vp], i32),
        "atkg_dataset_write_file_device": ([C.c_char_p, vp, u64, u64, vp], i32),
        "atkg_mips_score": ([vp, u64, vp, u64, u64, vp, u64, u64, vp], i32),
        "atkg_synth_distinct": ([u64, u64, u64, u64, vp, u32], i32),
        "atkg_synth_distinct_device": ([u64, u64, u64, u64, vp, vp], i32),
        "atkg_simulate_recall_many": ([P, u32, u64, u64, u32, f64p, f64p, vp], i32),
        "atkg_fill_normal": ([u64, u64, C.c_float, C.c_float, vp, u32], None),
        "atkg_fill_normal_range": ([u64, u64, u64, C.c_float, C.c_float, vp, u32], None),
        "atkg_f32_to_bf16": ([vp, u64, vp, u32], None),
        "atkg_bf16_to_f32": ([vp, u64, vp, u32], None),
        "atkg_profile_begin": ([], None),
        "atkg_profile_begin_every": ([C.c_uint32], None),
        "atkg_profile_end": ([f64p, C.POINTER(C.c_uint64)], i32),
        "atkg_launch_count": ([], u64),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def check(rc: int) -> None:
    """Maps an atkg status code to the reference's exception types."""
    if rc == ATKG_OK:
        return
    msg = lib.atkg_last_error().decode()
    if rc in (ATKG_EINVAL, ATKG_ENAN):
        raise ValueError(msg)
    if rc == ATKG_EINFEASIBLE:
        raise NoFeasibleConfigError(msg)
    if rc == ATKG_EFORMAT:
        raise DatasetFormatError(msg)
    if rc == ATKG_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def set_option(name: str, value: int | None) -> None:
    """Path-selection override (atkg_set_option); None restores the default."""
    check(lib.atkg_set_option(name.encode(), 2**64 - 1 if value is None else int(value)))


class option:
    """Context manager: `with option("st_force_slow", 1): ...` (tests)."""

    def __init__(self, name: str, value: int):
        self.name, self.value = name, value

    def __enter__(self):
        self.prev = lib.atkg_get_option(self.name.encode(), 2**64 - 1)
        set_option(self.name, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.name, None if self.prev == 2**64 - 1 else self.prev)


def make_params(n: int, num_buckets: int, local_k: int, global_k: int, lane_multiple: int = 128) -> Params:
    return Params(n, num_buckets, local_k, global_k, lane_multiple)
