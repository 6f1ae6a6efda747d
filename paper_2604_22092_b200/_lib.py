"""ctypes binding of libflashspread_b200.so (include/flashspread.h).

The structures below mirror the C layouts field for field (natural C
alignment, which ctypes reproduces).  Every call goes through `check`, which
turns a negative return code into the Python exception the reference would
raise.  There is no fallback: if the shared library or a CUDA device is
missing, importing the engine raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import FlashSpreadNativeError, InvalidConfigError, ReconfigureAfterStartError

MAX_COMPARTMENTS = 16
ABI_VERSION = 6

# enum fs_dtype
I8, I32, I64, F16, BF16, F32, F64, U32, U64 = 1, 2, 3, 4, 5, 6, 7, 8, 9
# enum fs_strategy
PER_NODE, LANE, MERGE, AUTO = 0, 1, 2, 3
# enum fs_hazard
HZ_NONE, HZ_EXPONENTIAL, HZ_LOGNORMAL, HZ_WEIBULL, HZ_ERLANG = 0, 1, 2, 3, 4
# enum fs_shedding
SHED_CONSTANT, SHED_LN_HAZARD, SHED_DENSITY_PEAK = 0, 1, 2
# enum fs_rng
RNG_SPLITMIX, RNG_PHILOX = 0, 1
# enum fs_hazard_precision
HAZ_F64, HAZ_F32 = 0, 1

FS_EINVAL, FS_ECUDA, FS_ENOMEM, FS_ESTATE, FS_ECONSERVE, FS_EREPR = -1, -2, -3, -4, -5, -6
FS_BUF_FRESH = 4  # fs_state_buffers.padded flag: a fresh state

_c_i32, _c_i64, _c_u64, _c_f32, _c_f64, _vp = (
    ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_double, ctypes.c_void_p,
)


class FsGraph(ctypes.Structure):
    _fields_ = [
        ("num_nodes", _c_i64),
        ("num_edges", _c_i64),
        ("row_offsets", _vp),
        ("row_offsets32", _vp),
        ("col_indices", _vp),
        ("weights", _vp),
        ("weights_dtype", _c_i32),
        ("weights_uniform", _c_i32),
        ("uniform_weight", _c_f32),
        ("d_max", _c_i32),
        ("padded", _c_i32),
        ("out_row_offsets", _vp),
        ("out_col_indices", _vp),
    ]


class FsCompartment(ctypes.Structure):
    _fields_ = [
        ("succ", _c_i32),
        ("terminal", _c_i32),
        ("hazard", _c_i32),
        ("pad_", _c_i32),
        ("p0", _c_f64),
        ("p1", _c_f64),
    ]


class FsModel(ctypes.Structure):
    _fields_ = [
        ("num_compartments", _c_i32),
        ("edge_from", _c_i32),
        ("edge_to", _c_i32),
        ("infectious", _c_i32),
        ("beta", _c_f64),
        ("shedding", _c_i32),
        ("pad_", _c_i32),
        ("shed_mu", _c_f64),
        ("shed_sigma", _c_f64),
        ("shed_peak", _c_f64),
        ("comp", FsCompartment * MAX_COMPARTMENTS),
    ]


class FsConfig(ctypes.Structure):
    _fields_ = [
        ("epsilon", _c_f64),
        ("tau_max", _c_f64),
        ("delta", _c_f64),
        ("steps_per_batch", _c_i32),
        ("strategy", _c_i32),
        ("compaction", _c_i32),
        ("mixed_precision", _c_i32),
        ("lanes_per_node", _c_i32),
        ("edges_per_block", _c_i32),
        ("hazard_chunk", _c_i32),
        ("chunk_skip", _c_i32),
        ("carry_tau", _c_i32),
        ("rng", _c_i32),
        ("hazard_precision", _c_i32),
        ("count_gather", _c_i32),
        ("incremental", _c_i32),
    ]


class FsScalars(ctypes.Structure):
    _fields_ = [
        ("clock", _c_f64),
        ("tau_next", _c_f64),
        ("step", _c_i64),
        ("seed", _c_u64),
        ("last_max_rate", _c_f32),
        ("started", _c_i32),
        ("counts", _c_i64 * MAX_COMPARTMENTS),
    ]


class FsStateBuffers(ctypes.Structure):
    _fields_ = [
        ("states", _vp),
        ("ages", _vp),
        ("infectivity", _vp * 2),
        ("imask", _vp * 2),
        ("pressure", _vp),
        ("rates", _vp),
        ("padded", _c_i32),
    ]


class FsPartition(ctypes.Structure):
    _fields_ = [
        ("node_base", _c_i64),
        ("num_nodes_global", _c_i64),
        ("mask_segment_words", _c_i64),
        ("rank", _c_i32),
        ("world", _c_i32),
        ("comm", _vp),
        ("range_bounds", _vp),
    ]


class FsMarkovConfig(ctypes.Structure):
    _fields_ = [("theta", _c_f64), ("p_max", _c_f64), ("tau_max", _c_f64), ("steps_per_batch", _c_i32),
                ("pad_", _c_i32)]


_SIGNATURES = {
    "fs_abi_version": (_c_i32, []),
    "fs_last_error": (ctypes.c_char_p, []),
    "fs_device_sm_count": (_c_i32, [_c_i32]),
    "fs_host_register": (_c_i32, [_vp, _c_i64]),
    "fs_host_unregister": (_c_i32, [_vp]),
    "fs_engine_create": (_c_i32, [ctypes.POINTER(FsGraph), ctypes.POINTER(FsModel), ctypes.POINTER(FsConfig),
                                   ctypes.POINTER(FsStateBuffers), ctypes.POINTER(FsScalars), _c_i32,
                                   ctypes.POINTER(_vp)]),
    "fs_engine_create_partitioned": (_c_i32, [ctypes.POINTER(FsGraph), ctypes.POINTER(FsModel),
                                              ctypes.POINTER(FsConfig), ctypes.POINTER(FsStateBuffers),
                                              ctypes.POINTER(FsScalars), _c_i32, ctypes.POINTER(FsPartition),
                                              ctypes.POINTER(_vp)]),
    "fs_engines_exchange_local": (_c_i32, [_vp, _c_i32, _vp]),
    "fs_engine_delta_buffers": (_c_i32, [_vp, _vp]),
    "fs_engine_acc_get": (_c_i32, [_vp, _vp, _vp]),
    "fs_engine_acc_set": (_c_i32, [_vp, _vp, _vp]),
    "fs_engine_reset_age_memo": (_c_i32, [_vp, _vp]),
    "fs_engine_states_edited": (_c_i32, [_vp, _vp]),
    "fs_engine_set_peer_deltas": (_c_i32, [_vp, _vp]),
    "fs_engine_mailbox": (_c_i32, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_c_i64)]),
    "fs_engine_set_peer_mailboxes": (_c_i32, [_vp, _vp]),
    "fs_engine_apply_mailbox": (_c_i32, [_vp, _vp]),
    "fs_ipc_get_handle": (_c_i32, [_vp, _vp, _c_i32]),
    "fs_ipc_open_handle": (_c_i32, [_vp, _c_i32, ctypes.POINTER(_vp)]),
    "fs_ipc_close": (_c_i32, [_vp]),
    "fs_comm_unique_id": (_c_i32, [_vp, _c_i32]),
    "fs_comm_init": (_c_i32, [_c_i32, _c_i32, _vp, _c_i32, ctypes.POINTER(_vp)]),
    "fs_comm_destroy": (None, [_vp]),
    "fs_engine_destroy": (None, [_vp]),
    "fs_markov_create": (_c_i32, [ctypes.POINTER(FsGraph), ctypes.POINTER(FsModel), ctypes.POINTER(FsMarkovConfig),
                                  _vp, _vp, ctypes.POINTER(FsScalars), _c_i32, ctypes.POINTER(_vp)]),
    "fs_markov_destroy": (None, [_vp]),
    "fs_markov_step": (_c_i32, [_vp, _c_i32, _vp]),
    "fs_markov_run_batch": (_c_i32, [_vp, _vp]),
    "fs_markov_get_scalars": (_c_i32, [_vp, ctypes.POINTER(FsScalars), _vp]),
    "fs_markov_set_scalars": (_c_i32, [_vp, ctypes.POINTER(FsScalars), _vp]),
    "fs_markov_read_log": (_c_i32, [_vp, _c_i64, _c_i32, _vp, _vp, _vp, _vp]),
    "fs_markov_influence": (_c_i32, [_vp, _vp, _vp]),
    "fs_markov_refresh_rates": (_c_i32, [_vp, _vp]),
    "fs_engine_uses_count_gather": (_c_i32, [_vp]),
    "fs_engine_kernels_per_step": (_c_i32, [_vp]),
    "fs_engine_sync_ages": (_c_i32, [_vp, _vp]),
    "fs_engine_state_restored": (_c_i32, [_vp, _vp]),
    "fs_seed_select": (_c_i32, [ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64, _vp, ctypes.c_int32, ctypes.c_int32,
                                _vp, ctypes.c_int32, ctypes.c_float, _vp, _vp]),
    "fs_seed_select_batch": (_c_i32, [ctypes.c_int64, ctypes.c_int32, _vp, ctypes.c_int64, _vp, ctypes.c_int64,
                                      ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int32, ctypes.c_float, _vp]),
    "fs_flags_to_ids": (_c_i32, [_vp, ctypes.c_int64, _vp, ctypes.POINTER(ctypes.c_int64), _vp]),
    "fs_check_symmetric": (_c_i32, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int32),
                                    _vp]),
    "fs_narrow_offsets": (_c_i32, [_vp, ctypes.c_int64, _vp, _vp]),
    "fs_fill": (_c_i32, [_vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, _vp]),
    "fs_engine_wait_log": (_c_i32, [_vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp, _vp]),
    "fs_engine_read_remote_pushes": (_c_i32, [_vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp]),
    "fs_comm_time_exchange": (_c_i32, [_vp, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, _vp,
                                       ctypes.POINTER(ctypes.c_float)]),
    "fs_h2d_staged": (_c_i32, [_vp, _vp, ctypes.c_int64, _vp]),
    "fs_host_csr_scan": (_c_i32, [_vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                  ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_float)]),
    "fs_engine_uniform_s_age": (_c_i32, [_vp]),
    "fs_ensemble_create": (_c_i32, [_vp, _c_i32, ctypes.POINTER(_vp)]),
    "fs_ensemble_destroy": (None, [_vp]),
    "fs_ensemble_grid": (_c_i32, [_vp, ctypes.POINTER(_c_i32)]),
    "fs_ensemble_run_batch": (_c_i32, [_vp, _vp]),
    "fs_ensemble_wait_log": (_c_i32, [_vp, _c_i64, _c_i32, _vp, _vp, _vp]),
    "fs_engine_current_buffer": (_c_i32, [_vp, _vp]),
    "fs_engine_begin_batch": (_c_i32, [_vp, _vp]),
    "fs_engine_step": (_c_i32, [_vp, _c_i32, _c_i32, _c_i32, _vp]),
    "fs_engine_run_batch": (_c_i32, [_vp, _c_i32, _vp]),
    "fs_engine_read_log": (_c_i32, [_vp, _c_i64, _c_i32, _vp, _vp, _vp, _vp]),
    "fs_engine_get_scalars": (_c_i32, [_vp, ctypes.POINTER(FsScalars), _vp]),
    "fs_engine_set_scalars": (_c_i32, [_vp, ctypes.POINTER(FsScalars), _vp]),
    "fs_engine_load_infectivity": (_c_i32, [_vp, _vp, _vp]),
    "fs_engine_store_infectivity": (_c_i32, [_vp, _vp, _vp]),
    "fs_pressure_gather": (_c_i32, [ctypes.POINTER(FsGraph), _vp, _c_i32, _vp, _c_i32, _c_i32, _c_i32, _vp]),
    "fs_uniform_fill": (_c_i32, [_c_u64, _c_u64, _vp, _c_i64, _c_i32, _vp, _vp]),
    "fs_hazard_eval": (_c_i32, [ctypes.POINTER(FsCompartment), _vp, _c_i64, _vp, _c_i32, _vp]),
    "fs_erfcx_eval": (_c_i32, [_vp, _c_i64, _vp, _vp]),
    "fs_gen_regular": (_c_i32, [_c_i64, _c_i32, _c_u64, _c_i64, _c_i64, _vp, _vp, _c_i64, ctypes.POINTER(_c_i64), _vp]),
    "fs_gen_barabasi_albert": (_c_i32, [_c_i64, _c_i32, _c_u64, _c_i64, _c_i64, _vp, _vp, _c_i64,
                                        ctypes.POINTER(_c_i64), _vp]),
    "fs_gen_erdos_renyi": (_c_i32, [_c_i64, _c_f64, _c_u64, _c_i64, _c_i64, _vp, _vp, _c_i64,
                                    ctypes.POINTER(_c_i64), _vp]),
    "fs_gen_regular_row_host": (_c_i32, [_c_i64, _c_i32, _c_u64, _c_i64, _vp]),
    "fs_refresh_active": (_c_i32, [_vp, _c_i32, _c_i64, _vp, _c_i32, _vp, _c_i64, ctypes.POINTER(_c_i64), _vp]),
    "fs_traj_records": (_c_i32, [_vp, _vp, _vp, _c_i64, _c_i64, _c_i32, _vp, _c_i32, _c_i64, _c_i32, _c_i32, _vp,
                                 _vp, _vp]),
    "fs_ensemble_mean": (_c_i32, [_vp, _c_i64, _c_i64, _vp, _vp]),
    "fs_column_quantiles": (_c_i32, [_vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i32, _vp, _vp, _vp, _vp, _vp]),
    "fs_bootstrap_metrics": (_c_i32, [_vp, _c_i64, _vp, _c_i64, _c_i32, _c_i32, _vp, _vp, _c_i64, _c_i32, _c_i32,
                                      _vp, _vp, _vp, _vp, _vp]),
    "fs_run_deviation": (_c_i32, [_vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_f64, _c_f64, _vp, _vp, _vp]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

# FS_LIB_PATH selects another build of the same ABI (A/B measurements only)
LIB_PATH = Path(os.environ.get("FS_LIB_PATH") or Path(__file__).resolve().parent / "libflashspread_b200.so")
_lib = None


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise FlashSpreadNativeError(
            f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        if os.environ.get("FS_LIB_PATH") and not hasattr(lib, name):
            continue  # an older build under A/B measurement
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.fs_abi_version() != ABI_VERSION:
        raise FlashSpreadNativeError(f"ABI version mismatch: {lib.fs_abi_version()} != {ABI_VERSION}")
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> int:
    """Map a C return code onto the reference's exception types."""
    if rc >= 0:
        return rc
    msg = load().fs_last_error().decode(errors="replace")
    if rc == FS_EINVAL:
        raise InvalidConfigError(msg)
    if rc == FS_ESTATE:
        raise ReconfigureAfterStartError(msg)
    if rc == FS_ECONSERVE:
        raise AssertionError(msg)
    raise FlashSpreadNativeError(f"libflashspread_b200 error {rc}: {msg}")


def ptr(t) -> int | None:
    """Raw device address of a torch tensor (None for empty / missing)."""
    if t is None or t.numel() == 0:
        return None
    return t.data_ptr()
