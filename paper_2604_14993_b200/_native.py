"""ctypes binding of libchainserve_b200.so (include/chainserve_b200.h).

The engine has no CPU fallback: if the shared library is missing or no CUDA
device is visible, every compute call raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import InfeasibleError, UnstableError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libchainserve_b200.so")

CS_OK, CS_INFEASIBLE, CS_INVALID, CS_INTERNAL, CS_ERR_CUDA, CS_UNSUPPORTED, CS_UNSTABLE = range(7)
CS_STREAMS_WHOLE_SM = 1
CS_SIM_PREFIX_READY = 1
CS_SIM_STREAMS_IL4 = 4
CS_SIM_FORCE_EVENT_LOOP = 2


class NativeUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library not built or no GPU)."""


class SimPoint(C.Structure):
    _fields_ = [("n_chains", C.c_int32), ("chain_base", C.c_int32), ("lam", C.c_double)]


class RepSummary(C.Structure):
    _fields_ = [
        ("wait_sum", C.c_double), ("service_sum", C.c_double), ("counted", C.c_int64),
        ("window_s", C.c_double), ("mean_occupancy", C.c_double),
        ("occ_first_half", C.c_double), ("occ_second_half", C.c_double),
        ("lambda_effective", C.c_double), ("end_queue_len", C.c_int64),
        ("w_start", C.c_double), ("t_mid", C.c_double), ("area_mid", C.c_double),
        ("t_end", C.c_double), ("area_end", C.c_double), ("resp_sum", C.c_double),
        ("resp_mean", C.c_double),
    ]


class ComposePoint(C.Structure):
    _fields_ = [
        ("n_servers", C.c_int32), ("server_base", C.c_int32), ("block_count", C.c_int64),
        ("block_bytes", C.c_int64), ("cache_slot_bytes", C.c_int64), ("capacity", C.c_int64),
        ("arrival_rate", C.c_double), ("load_target", C.c_double),
    ]


class BoundPoint(C.Structure):
    _fields_ = [("n_chains", C.c_int32), ("chain_base", C.c_int32), ("lam", C.c_double)]


class BdPoint(C.Structure):
    _fields_ = [("n_states", C.c_int32), ("base", C.c_int32), ("lam", C.c_double),
                ("total_rate", C.c_double)]


BOUNDS_DTYPE = np.dtype([("lower_occupancy", "<f8"), ("upper_occupancy", "<f8"),
                         ("lower_response_s", "<f8"), ("upper_response_s", "<f8"),
                         ("total_rate", "<f8"), ("total_capacity", "<i4"), ("status", "<i4")])

SUMMARY_DTYPE = np.dtype([(name, np.float64 if ct is C.c_double else np.int64)
                          for name, ct in RepSummary._fields_])
assert SUMMARY_DTYPE.itemsize == C.sizeof(RepSummary)

EXPORTS = (
    "cs_version", "cs_last_error", "cs_host_log1p_variant", "cs_device_count", "cs_launch_count",
    "cs_release_memory",
    "cs_philox_keys", "cs_exp_streams", "cs_jffc_sim", "cs_jffc_sim_workspace_bytes", "cs_seg_plan", "cs_philox_peak", "cs_sim_streams", "cs_sim_streams_ex", "cs_jffc_sim_ex",
    "cs_rep_stats", "cs_rep_stats_dist", "cs_run_sim_host", "cs_gbp_batch", "cs_gca_batch",
    "cs_nccl_unique_id", "cs_comm_init", "cs_comm_destroy", "cs_occupancy_bounds",
    "cs_birth_death_occupancy", "cs_sim_ext", "cs_ragged_rows",
)

_lib = None


def load(require_device: bool = True):
    """Load the library (building it first if it is absent and nvcc exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            try:
                from .build import build
                build()
            except Exception as exc:  # pragma: no cover - depends on toolchain
                raise NativeUnavailable(f"libchainserve_b200.so missing and build failed: {exc}")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        vp = C.c_void_p
        L.cs_version.restype = C.c_char_p
        L.cs_last_error.restype = C.c_char_p
        L.cs_launch_count.restype = C.c_int64
        L.cs_philox_keys.argtypes = [P(C.c_uint32), C.c_int32, P(C.c_uint64), C.c_int64, P(C.c_uint64)]
        L.cs_exp_streams.argtypes = [vp, C.c_int64, C.c_int64, vp, C.c_int64, C.c_int32, vp]
        L.cs_jffc_sim.argtypes = [vp, C.c_int32, vp, vp, C.c_int32, C.c_int32, vp, C.c_int64,
                                  C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int64, vp,
                                  C.c_int64, vp, C.c_int32, vp, vp, vp, C.c_int64, vp]
        L.cs_jffc_sim_workspace_bytes.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                  C.c_int64]
        L.cs_jffc_sim_workspace_bytes.restype = C.c_int64
        L.cs_seg_plan.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int64, P(C.c_int32)]
        L.cs_philox_peak.argtypes = [C.c_int64, C.c_int32, vp, vp]
        L.cs_jffc_sim_ex.argtypes = L.cs_jffc_sim.argtypes[:-1] + [C.c_int32, vp]
        L.cs_sim_streams.argtypes = [vp, C.c_int64, C.c_int64, vp, C.c_int64, C.c_int32, vp, C.c_int32,
                                     C.c_int32, C.c_int32, C.c_int64, C.c_int64, vp, C.c_int64,
                                     P(C.c_int32), vp]
        L.cs_sim_streams_ex.argtypes = L.cs_sim_streams.argtypes[:-2] + [C.c_int32, P(C.c_int32), vp]
        L.cs_rep_stats.argtypes = [vp, C.c_int32, C.c_int64, C.c_int64, C.c_int64, vp,
                                   P(C.c_int64), C.c_int32, P(C.c_double), vp, vp]
        L.cs_rep_stats_dist.argtypes = L.cs_rep_stats.argtypes
        L.cs_nccl_unique_id.argtypes = [C.c_char_p]
        L.cs_comm_init.argtypes = [C.c_char_p, C.c_int32, C.c_int32]
        L.cs_run_sim_host.argtypes = [
            P(SimPoint), C.c_int32, P(C.c_double), P(C.c_int32), C.c_int32, P(C.c_uint32),
            C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int64, P(C.c_int64), C.c_int32,
            C.c_int32, C.c_int64, vp, P(C.c_double), C.c_int32, P(C.c_double), P(C.c_double),
            P(C.c_double), vp]
        L.cs_gbp_batch.argtypes = [vp, C.c_int32, C.c_int32] + [vp] * 14 + [vp]
        L.cs_gca_batch.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32] + [vp] * 7 + \
            [C.c_int32, C.c_int32] + [vp] * 7 + [vp]
        L.cs_occupancy_bounds.argtypes = [vp, C.c_int32, vp, vp, C.c_int32, vp, vp, vp]
        L.cs_birth_death_occupancy.argtypes = [vp, C.c_int32, vp, C.c_int32, vp, vp, vp]
        L.cs_sim_ext.argtypes = [vp, vp]
        L.cs_ragged_rows.argtypes = [vp, C.c_int32, C.c_int64, vp, vp, vp]
        _lib = L
    if require_device and _lib.cs_device_count() == 0:
        raise NativeUnavailable("no CUDA device visible: the chainserve B200 engine has no CPU path")
    return _lib


def last_error() -> str:
    return (load(False).cs_last_error() or b"").decode()


def check(status: int, what: str) -> None:
    if status == CS_OK:
        return
    msg = f"{what}: {last_error()}"
    if status == CS_INFEASIBLE:
        raise InfeasibleError(msg)
    if status == CS_INVALID:
        raise ValueError(msg)
    if status == CS_INTERNAL:
        raise AssertionError(msg)
    if status == CS_UNSUPPORTED:
        raise NotImplementedError(msg)
    if status == CS_UNSTABLE:
        raise UnstableError(msg)
    raise NativeUnavailable(msg)


def ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def seed_words(seed: int) -> np.ndarray:
    """numpy _coerce_to_uint32_array(seed): little-endian uint32 words."""
    if seed < 0:
        raise ValueError("expected non-negative integer")
    words = []
    if seed == 0:
        words.append(0)
    while seed > 0:
        words.append(seed & 0xFFFFFFFF)
        seed >>= 32
    return np.asarray(words, dtype=np.uint32)


def seg_plan(n_points: int, n_reps: int, max_capacity: int, n_jobs: int) -> dict:
    """Launch plan of the segmented single-chain simulator for this shape."""
    out = (C.c_int32 * 4)()
    check(load().cs_seg_plan(n_points, n_reps, max_capacity, n_jobs, out), "cs_seg_plan")
    return {"segments": out[0], "warps_per_segment": out[1], "checkpoints": out[2], "cmax": out[3]}
