"""ctypes binding of libtinymd_b200.so (the C ABI in include/tinymd_b200.h).

Loaded eagerly at import so a missing or stale library fails loudly; there is
no CPU fallback anywhere in the package.  Device pointers come from torch
tensors (``tensor.data_ptr()``); every call is enqueued on the caller's
current torch CUDA stream.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import GuardViolation, NativeError, ProtocolError, SingularityError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtinymd_b200.so")

OK, CAPACITY, PROTOCOL, SINGULARITY, GUARD, ERR_CUDA, ERR_ARG = range(7)
F_ENERGY, F_EXACT, F_STORE_FORCES, F_NO_PRUNE, F_SKIP_FORCES = 1, 2, 4, 8, 16
SEL_GE, SEL_LT, SEL_GT, SEL_IN = 0, 1, 2, 3
STATUS_WORDS = 4

_p, _i32, _i64, _u32, _f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_double

# name -> argtypes (restype is int for all but tmd_last_error)
SIGNATURES = {
    "tmd_version": [],
    "tmd_device_info": [_p, _p, _p, _p],
    "tmd_status_reset": [_p, _p],
    "tmd_bin_cells": [_p, _i64, _i32, _p, _f64, _p, _p, _p, _p, _p, _p],
    "tmd_build_lists": [_p, _i64, _i32, _p, _p, _p, _p, _i64, _p, _f64, _i32, _i32, _p, _i64, _p, _p, _p],
    "tmd_cell_positions": [_p, _i64, _p, _i32, _p, _i64, _p],
    "tmd_permute_rows": [_p, _i64, _p, _i32, _p, _i64, _i32, _p],
    "tmd_force_lj": [_p, _i64, _i32, _p, _i64, _p, _i32, _f64, _f64, _f64, _u32, _p, _i64, _p,
                     _p, _p],
    "tmd_force_sd": [_p, _p, _i64, _i32, _p, _i64, _p, _i32, _f64, _f64, _f64, _u32, _p, _i64,
                     _p, _p, _p],
    "tmd_force_half": [_p, _p, _i64, _i32, _p, _i64, _p, _i32, _f64, _f64, _f64, _u32, _p, _i64,
                       _p, _p, _p],
    "tmd_step_lj": [_p, _p, _p, _i64, _i32, _p, _i64, _p, _p, _i32, _f64, _p, _p, _p, _p, _p, _i64, _i32, _p,
                    _p, _p, _f64, _f64, _f64, _f64, _f64, _i32, _u32, _p, _i64, _p, _i64, _p, _p, _p, _f64, _p],
    "tmd_step_sd": [_p, _p, _p, _p, _i64, _i32, _p, _i64, _p, _p, _i32, _f64, _p, _p, _p, _p, _p, _i64, _i32, _p,
                    _p, _p, _f64, _f64, _f64, _f64, _f64, _i32, _u32, _p, _i64, _p, _i64, _p, _p, _p, _f64, _p],
    "tmd_zero_rows": [_p, _i64, _i32, _i64, _i64, _p],
    "tmd_compose_inverse": [_p, _p, _i32, _p, _p],
    "tmd_group_by_rank": [_p, _p, _i32, _i32, _p, _p, _p, _p],
    "tmd_peer_allgather": [_i64, _i32, _i32, _p, _p, _i32, _p, _f64, _p, _p],
    "tmd_sort_locals": [_p, _p, _i64, _i32, _p, _f64, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
    "tmd_run_steps": [_p, _i32, _i32, _p],
    "tmd_epoch_p1": [_p, _p],
    "tmd_run_launch_times": [_p, _p, _i32],
    "tmd_pack_rows": [_p, _p, _i64, _p, _i32, _i32, _p, _p],
    "tmd_unpack_rows": [_p, _i32, _i32, _p, _p, _i64, _i32, _p],
    "tmd_border_slots": [_p, _i32, _i32, _p, _p, _p],
    "tmd_gather_i32": [_p, _p, _i32, _p, _p],
    "tmd_sfc_keys": [_p, _i64, _i32, _p, _p, _i32, _i32, _p, _p],
    "tmd_leaf_counts": [_p, _i32, _p, _i32, _p, _p],
    "tmd_check_pack": [_p, _p, _i32, _p, _p],
    "tmd_copy_rows": [_p, _i64, _p, _i64, _i32, _i64, _p],
    "tmd_exports_build": [_i32, _i32, _p, _p, _p, _p, _i64, _p, _p, _p, _p, _p, _p],
    "tmd_ghost_provenance": [_i32, _i32, _i32, _p, _i32, _p, _p, _p, _p, _i64, _p, _p, _p, _i64, _p],
    "tmd_ipc_handle": [_p, _p, _p],
    "tmd_brick_sort": [_p, _i64, _i32, _p, _f64, _p, _p, _p, _p, _p, _p],
    "tmd_mailbox_words": [],
    "tmd_peer_gather_words": [],
    "tmd_prepare_stream": [_p],
    "tmd_peer_sync": [_i64, _i32, _i32, _p, _p, _f64, _p, _p],
    "tmd_borders_count": [_p, _i64, _i32, _p, _p, _p, _p],
    "tmd_borders_fill": [_p, _i64, _i32, _p, _p, _p, _p, _p, _p, _p, _i64, _p, _p, _p, _i64, _p, _p],
    "tmd_exchange_classify": [_p, _i64, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
    "tmd_ipc_open": [_p, _i64, _p, _p],
    "tmd_ipc_close": [_p],
    "tmd_ipc_handle_size": [],
    "tmd_build_lists_split": [_p, _i64, _i32, _p, _p, _p, _p, _i64, _p, _f64, _p, _i32, _f64, _p, _f64, _i32, _p,
                              _i64, _p, _p, _p, _p, _p],
    "tmd_split_margin": [_p, _i32, _i32, _f64, _f64, _f64, _f64, _p, _p],
    "tmd_bin_cells_ex": [_p, _i64, _i32, _p, _f64, _p, _i32, _p, _p, _p, _p, _p],
    "tmd_bin_cells_dev": [_p, _i64, _i32, _i32, _p, _p, _f64, _p, _i32, _p, _p, _p, _p, _p],
    "tmd_cell_positions_dev": [_p, _i64, _p, _i32, _i32, _p, _p, _i64, _p, _p],
    "tmd_exports_build_dev": [_i32, _i32, _p, _p, _p, _p, _p, _i64, _p, _p, _p, _p, _i64, _p, _p],
    "tmd_borders_fill_capped": [_p, _i64, _i32, _p, _p, _p, _p, _p, _p, _p, _i64, _p, _p, _p, _i64, _p, _i64, _p],
    "tmd_kick_drift": [_p, _p, _p, _i64, _i64, _i32, _f64, _f64, _p, _i64, _p, _p],
    "tmd_kick": [_p, _p, _i64, _i64, _i32, _f64, _p],
    "tmd_max_disp2": [_p, _i64, _p, _i64, _i32, _p, _p],
    "tmd_kinetic": [_p, _i64, _i32, _f64, _p, _p],
    "tmd_select": [_p, _i32, _i32, _f64, _f64, _p, _p, _p],
    "tmd_select_pair": [_p, _i32, _i32, _f64, _i32, _f64, _p, _p, _p, _p],
    "tmd_emit_ghosts": [_p, _p, _i64, _p, _i32, _p, _i32, _i32, _p, _p],
    "tmd_gather_shift": [_p, _i64, _p, _i32, _p, _i32, _p, _p, _i64, _p],
    "tmd_plan_shift": [_p, _i64, _p, _i32, _i32, _f64, _p, _p],
    "tmd_wrap_self": [_p, _i64, _i32, _i32, _f64, _f64, _f64, _f64, _p],
    "tmd_check_owned": [_p, _i64, _i32, _p, _p, _p, _p],
    "tmd_sync_flat": [_p, _i64, _i32, _i32, _p, _p, _p],
    "tmd_flatten_round": [_i32, _i32, _i32, _p, _i32, _p, _p, _p, _i64, _p],
    "tmd_pair_force": [_i32, _p, _p, _p, _p, _i32, _f64, _f64, _f64, _p, _p],
    "tmd_pair_energy": [_i32, _p, _i32, _f64, _f64, _f64, _p, _p],
}


class StepRun(C.Structure):
    """TmdStepRun (include/tinymd_b200.h): the batched step loop's arguments."""

    _fields_ = [("law", _i64), ("pos_a", _p), ("pos_b", _p), ("vel_a", _p), ("vel_b", _p), ("ld", _i64),
                ("n_local", _i64), ("nbr", _p), ("ld_nbr", _i64), ("nnbr", _p), ("nnear", _p), ("cap", _i64),
                ("near_margin", _f64), ("dispmax2", _p), ("ex_start", _p), ("ex_rank", _p), ("ex_slot", _p),
                ("ex_sh", _p), ("n_ex", _i64), ("n_peers", _i64), ("peer_base0", _p), ("peer_base1", _p),
                ("peer_ld", _p), ("ex_border", _p), ("p0", _f64), ("p1", _f64), ("p2", _f64),
                ("half_dt_over_m", _f64), ("dt", _f64), ("frc", _p), ("ld_f", _i64), ("xref", _p),
                ("ld_ref", _i64), ("thermo", _p), ("thermo_stride", _i64), ("status", _p), ("guard_lim2", _f64),
                ("k_last", _i64), ("epoch_step", _i64), ("reneigh", _i64), ("thermo_every", _i64),
                ("store_every", _i64), ("rebuild_at_k0", _i64), ("barrier_epoch0", _i64), ("rank", _i64),
                ("size", _i64), ("mailboxes", _p), ("barrier_timeout_s", _f64), ("time_launches", _i64)]


_D3, _I3 = _f64 * 3, _i64 * 3


class EpochP1(C.Structure):
    """TmdEpochP1 (include/tinymd_b200.h): the P = 1 epoch's arguments."""

    _fields_ = [("pos", _p), ("pos_alt", _p), ("vel", _p), ("vel_alt", _p), ("ld", _i64), ("n", _i64),
                ("room", _i64), ("sd", _i64), ("wrap_hi", _D3), ("wrap_lo", _D3), ("wrap_s_plus", _D3),
                ("wrap_s_minus", _D3), ("slab_lo", _D3), ("slab_hi", _D3), ("sort_lo", _D3), ("sort_edge", _f64),
                ("sort_dims", _I3), ("sort_shell", _i64), ("sort_shape", _I3), ("sort_cell_of", _p),
                ("sort_cell_start", _p), ("sort_cell_atoms", _p), ("sort_key", _p), ("sort_key_start", _p),
                ("sort_perm", _p), ("order", _p), ("thr_hi", _D3), ("thr_lo", _D3), ("s_hi", _D3), ("s_lo", _D3),
                ("off", _p), ("root", _p), ("sh", _p), ("ld_sh", _i64), ("bin_lo", _D3), ("bin_edge", _f64),
                ("bin_dims", _I3), ("bin_shell", _i64), ("cell_of", _p), ("cell_start", _p), ("cell_atoms", _p),
                ("cell_pos", _p), ("ld_cp", _i64), ("cell_pos_f", _p), ("f32_eps", _f64), ("dispmax2", _p),
                ("margin_i0", _i64), ("margin_i1", _i64),
                ("margin_floor", _f64), ("margin_factor", _f64), ("margin_cap", _f64), ("cutoff", _f64),
                ("margin_out", _p), ("nbr", _p), ("ld_nbr", _i64), ("nnear", _p), ("counts", _p), ("cap", _i64),
                ("near_rsq", _f64), ("rsq_max", _f64), ("xref", _p), ("ld_ref", _i64), ("ex_start", _p),
                ("ex_rank", _p), ("ex_slot", _p), ("ex_sh", _p), ("ex_zeros", _p), ("ex_slots", _p), ("ld_o", _i64),
                ("status", _p), ("list_status", _p)]


def header_symbols() -> list[str]:
    """Every function the public header declares (tests check the .so exports them)."""
    import re

    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(here, "include", "tinymd_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|uint64_t|const char\*)\s+(tmd_\w+)\s*\(", text, re.M)))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2009_07400_b200/build.py` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.tmd_last_error.argtypes = []
    lib.tmd_last_error.restype = C.c_char_p
    lib.tmd_launch_count.argtypes = []
    lib.tmd_launch_count.restype = C.c_int64
    return lib


lib = _load()


def launch_count() -> int:
    """Kernels launched by libtinymd_b200.so so far in this process."""
    return int(lib.tmd_launch_count())


def check(rc: int, what: str) -> None:
    if rc != OK:
        msg = lib.tmd_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed with code {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args), name)


def host_f64(values) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(values, dtype=np.float64))


def host_i32(values) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(values, dtype=np.int32))


def hp(a: np.ndarray) -> int:
    """Host pointer of a contiguous numpy array (kept alive by the caller)."""
    return a.ctypes.data


def decode_status(words: np.ndarray):
    code = int(words[0])
    key = int(np.uint64(words[1]))
    need = int(words[2])
    return code, key, need


def raise_for_status(words, *, context: str = "", describe=None) -> None:
    """Map a device status word onto the reference's exception classes."""
    code, key, need = decode_status(np.asarray(words))
    if code == OK:
        return
    detail = describe(code, key) if describe else ""
    if code == PROTOCOL:
        raise ProtocolError(f"{context}: protocol violation at atom {key}{detail}")
    if code == SINGULARITY:
        i, k = key >> 32, key & 0xFFFFFFFF
        raise SingularityError(f"{context}: coincident pair: local {i} (list slot {k}){detail}")
    if code == GUARD:
        raise GuardViolation(f"{context}{detail}")
    if code == CAPACITY:
        raise NativeError(f"{context}: neighbor capacity {need} needed (unhandled)")
    raise NativeError(f"{context}: device status {code}")
