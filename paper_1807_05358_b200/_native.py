"""ctypes binding of libparasim_cuda.so (include/parasim.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is usable, every entry point raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["lib", "NativeUnavailable", "check", "PsProblemDesc", "PsProblemInfo", "PsTraceTask",
           "PsMcmcParams", "PsChainSummary", "LIB_PATH", "ptr"]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PARASIM_B200_LIB") or os.path.join(HERE, "_lib", "libparasim_cuda.so")

PS_OK, PS_ERR_INVALID, PS_ERR_NO_ROUTE, PS_ERR_CYCLE, PS_ERR_CAPACITY, PS_ERR_CUDA = range(6)
PS_STATUS_OK, PS_STATUS_NO_ROUTE, PS_STATUS_CAPACITY, PS_STATUS_STOPPED = 0, 2, 4, 9
PS_HOST_PTRS, PS_DEVICE_PTRS = 0, 1
PS_RNG_PHILOX, PS_RNG_MT19937 = 0, 1
ABI_VERSION = 3

c_int_p = ctypes.POINTER(ctypes.c_int32)
c_i64_p = ctypes.POINTER(ctypes.c_int64)
c_dbl_p = ctypes.POINTER(ctypes.c_double)


class NativeUnavailable(RuntimeError):
    pass


class PsProblemDesc(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("n_ops", ctypes.c_int32), ("n_devices", ctypes.c_int32), ("n_kinds", ctypes.c_int32),
        ("n_links", ctypes.c_int32), ("n_pairs", ctypes.c_int32), ("n_maps", ctypes.c_int32),
        ("mode_full", ctypes.c_int32), ("n_slots", ctypes.c_int32), ("ready_capacity", ctypes.c_int32),
        ("dev_kind", c_int_p), ("link_of", c_int_p), ("link_bw", c_dbl_p), ("link_lat", c_dbl_p),
        ("op_ndim", c_int_p), ("op_dim", c_i64_p), ("op_esize", c_int_p), ("op_param_mask", c_int_p),
        ("op_map_off", c_int_p), ("op_nmaps_enum", c_int_p), ("op_slot_off", c_int_p), ("slot_op", c_int_p),
        ("op_in_off", c_int_p), ("op_in_pairs", c_int_p), ("op_out_off", c_int_p), ("op_out_pairs", c_int_p),
        ("map_deg", c_int_p), ("map_size", c_int_p), ("exe_fwd", c_dbl_p), ("exe_bwd", c_dbl_p),
        ("map_shard", c_dbl_p), ("map_ngroups", c_int_p),
        ("pair_src", c_int_p), ("pair_dst", c_int_p), ("pair_need_off", c_int_p), ("need", c_int_p),
        ("combo_off", c_int_p), ("combo_row_off", c_int_p), ("combo_col_off", c_int_p),
        ("backward_multiplier", ctypes.c_double),
    ]


class PsProblemInfo(ctypes.Structure):
    _fields_ = [("n_entries", ctypes.c_int64), ("n_combos", ctypes.c_int64), ("n_queues", ctypes.c_int32),
                ("n_slots", ctypes.c_int32), ("ready_capacity", ctypes.c_int32),
                ("warps_per_block", ctypes.c_int32), ("device_bytes", ctypes.c_int64),
                ("shared_counters", ctypes.c_int32), ("resident_warps_per_sm", ctypes.c_int32),
                ("smem_per_block", ctypes.c_int32), ("reserved_", ctypes.c_int32)]


class PsTraceTask(ctypes.Structure):
    _fields_ = [("key", ctypes.c_uint64), ("queue", ctypes.c_int32), ("aux", ctypes.c_int32),
                ("exe", ctypes.c_double), ("nbytes", ctypes.c_double), ("ready", ctypes.c_double),
                ("start", ctypes.c_double), ("end", ctypes.c_double)]


TRACE_DTYPE = np.dtype([("key", np.uint64), ("queue", np.int32), ("aux", np.int32), ("exe", np.float64),
                        ("nbytes", np.float64), ("ready", np.float64), ("start", np.float64),
                        ("end", np.float64)])


class PsMcmcParams(ctypes.Structure):
    _fields_ = [("rng_mode", ctypes.c_int32), ("beta_given", ctypes.c_int32), ("beta", ctypes.c_double),
                ("ln10", ctypes.c_double), ("record_trace", ctypes.c_int32), ("trace_capacity", ctypes.c_int32),
                ("delta", ctypes.c_int32), ("reserved_", ctypes.c_int32)]

    def __init__(self, rng_mode=0, beta_given=0, beta=0.0, ln10=0.0, record_trace=0, trace_capacity=0, delta=1):
        super().__init__(rng_mode, beta_given, beta, ln10, record_trace, trace_capacity, delta, 0)


class PsChainSummary(ctypes.Structure):
    _fields_ = [("initial_cost", ctypes.c_double), ("best_cost", ctypes.c_double), ("cost", ctypes.c_double),
                ("beta", ctypes.c_double), ("proposals", ctypes.c_int64), ("accepted", ctypes.c_int64),
                ("status", ctypes.c_int32), ("err_a", ctypes.c_int32), ("err_b", ctypes.c_int32),
                ("last_op", ctypes.c_int32), ("rounds_run", ctypes.c_int64), ("rounds_reused", ctypes.c_int64)]


_lib = None
_load_error = None


def ptr(a: np.ndarray, ctype=ctypes.c_void_p):
    return a.ctypes.data_as(ctype) if ctype is not ctypes.c_void_p else ctypes.c_void_p(a.ctypes.data)


def lib():
    """The loaded library; raises NativeUnavailable when it cannot be used."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise NativeUnavailable(_load_error)
    if not os.path.exists(LIB_PATH):
        _load_error = (f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                       " (there is no CPU fallback)")
        raise NativeUnavailable(_load_error)
    L = ctypes.CDLL(LIB_PATH)
    vp = ctypes.c_void_p
    L.ps_last_error.restype = ctypes.c_char_p
    L.ps_abi_version.restype = ctypes.c_int
    L.ps_problem_create.argtypes = [ctypes.POINTER(PsProblemDesc), ctypes.c_int, ctypes.POINTER(vp)]
    L.ps_problem_destroy.argtypes = [vp]
    L.ps_problem_destroy.restype = None
    L.ps_problem_info_get.argtypes = [vp, ctypes.POINTER(PsProblemInfo)]
    L.ps_combo_entries.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp,
                                   ctypes.POINTER(ctypes.c_int)]
    L.ps_simulate_batch.argtypes = [vp, vp, vp, ctypes.c_int, vp, vp, ctypes.c_int, vp]
    L.ps_simulate_batch_ex.argtypes = [vp, vp, vp, ctypes.c_int, vp, vp, vp, ctypes.c_int, vp]
    L.ps_simulate_trace.argtypes = [vp, vp, vp, ctypes.c_int, vp, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                    vp, vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_int32), vp]
    L.ps_mcmc_create.argtypes = [vp, ctypes.POINTER(PsMcmcParams), ctypes.c_int, vp, vp, vp, vp,
                                 ctypes.POINTER(vp)]
    L.ps_mcmc_run.argtypes = [vp, ctypes.c_int, vp]
    L.ps_mcmc_run_budget.argtypes = [vp, ctypes.c_int, ctypes.c_uint64, vp]
    L.ps_mcmc_read.argtypes = [vp, vp, vp, vp, vp, vp]
    L.ps_delta_batch.argtypes = [vp, vp, vp, vp, ctypes.c_int, vp, vp, vp, ctypes.c_int, vp]
    L.ps_mcmc_stop.argtypes = [vp, vp]
    L.ps_mcmc_chains.argtypes = [vp]
    L.ps_mcmc_read_state.argtypes = [vp, vp, vp]
    L.ps_simulate_explicit.argtypes = [ctypes.c_int, ctypes.c_int] + [vp] * 9 + \
        [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32), ctypes.c_int]
    L.ps_mcmc_destroy.argtypes = [vp]
    L.ps_mcmc_destroy.restype = None
    L.ps_mcmc_best.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)]
    if L.ps_abi_version() != ABI_VERSION:
        _load_error = "libparasim_cuda.so ABI version mismatch; rebuild"
        raise NativeUnavailable(_load_error)
    _lib = L
    return L


def check(rc: int, what: str):
    if rc != PS_OK:
        msg = lib().ps_last_error().decode(errors="replace")
        if rc == PS_ERR_CUDA:
            raise NativeUnavailable(f"{what}: CUDA error: {msg}")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")
