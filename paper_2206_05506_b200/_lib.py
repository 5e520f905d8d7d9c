"""ctypes binding of the C ABI in include/pnce_b200.h (libpnce_b200.so).

There is no CPU fallback: importing the compute entry points without the
built library, or calling them without an sm_100 device, raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PNCE_LIB", os.path.join(_HERE, "lib", "libpnce_b200.so"))

PNCE_DTYPE_FP16 = 0
PNCE_DTYPE_BF16 = 1

_STATUS = {
    1: E.InvalidConfigError,
    2: E.InvalidSpecError,
    3: E.ZeroStateError,
    4: E.NotMaximalLengthError,
    5: E.DimensionMismatchError,
    6: E.FrameTooShortError,
    7: E.PlanMismatchError,
    8: E.RowsOutOfRangeError,
    9: E.SaturationDetectedError,
    10: E.DeviceError,
    11: E.DeviceError,
}

# Every symbol the header declares (checked by tests/test_abi.py).
EXPORTS = (
    "pnce_version", "pnce_last_error", "pnce_config_check", "pnce_generate_mseq",
    "pnce_plan_create", "pnce_plan_create_rows", "pnce_plan_destroy", "pnce_plan_chips", "pnce_plan_operand",
    "pnce_workspace_bytes",
    "pnce_pack_iq", "pnce_correlate", "pnce_process_frames", "pnce_process_frames_scored", "pnce_process_frames_gather",
    "pnce_process_frames_tensor16", "pnce_process_bodies_tensor16", "pnce_copy_bodies_h2d", "pnce_process_bodies", "pnce_draw_channel", "pnce_simulate_frames", "pnce_kernel_launches",
)


class CfgStruct(ctypes.Structure):
    """pnce_cfg_t."""

    _fields_ = [
        ("m", ctypes.c_int32), ("c", ctypes.c_int32), ("n_t", ctypes.c_int32),
        ("n_r", ctypes.c_int32), ("n_batch", ctypes.c_int32), ("l", ctypes.c_int32),
        ("degree", ctypes.c_int32), ("tap_mask", ctypes.c_uint32), ("state", ctypes.c_uint32),
        ("dtype", ctypes.c_int32),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libpnce_b200.so once; raise DeviceError if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise E.DeviceError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    u64, f64 = ctypes.c_uint64, ctypes.c_double
    cfgp = ctypes.POINTER(CfgStruct)
    sig = {
        "pnce_version": (i32, []),
        "pnce_last_error": (ctypes.c_char_p, []),
        "pnce_config_check": (i32, [cfgp]),
        "pnce_generate_mseq": (i32, [i32, ctypes.c_uint32, ctypes.c_uint32, vp, i32, vp]),
        "pnce_plan_create": (i32, [cfgp, ctypes.POINTER(vp), vp]),
        "pnce_plan_create_rows": (i32, [cfgp, vp, i32, i32, ctypes.POINTER(vp), vp]),
        "pnce_plan_destroy": (i32, [vp]),
        "pnce_plan_chips": (i32, [vp, vp, vp]),
        "pnce_plan_operand": (i32, [vp, vp, ctypes.POINTER(i32), ctypes.POINTER(i32), vp]),
        "pnce_workspace_bytes": (sz, [vp, i64]),
        "pnce_pack_iq": (i32, [vp, vp, vp, i64, vp]),
        "pnce_correlate": (i32, [vp, vp, vp, vp, vp, i64, vp]),
        "pnce_process_frames": (i32, [vp, vp, vp, vp, vp, vp, sz, i64, vp]),
        "pnce_process_frames_gather": (i32, [vp, vp, vp, vp, i32, i32, i32, i64, vp]),
        "pnce_process_frames_scored": (i32, [vp, vp, vp, vp, vp, vp, i64, vp]),
        "pnce_process_frames_tensor16": (i32, [vp, vp, vp, vp, vp, i32, i32, i64, vp]),
        "pnce_process_bodies_tensor16": (i32, [vp, vp, i32, vp, vp, vp, i32, i32, i64, vp]),
        "pnce_copy_bodies_h2d": (i32, [vp, vp, vp, i32, i64, vp]),
        "pnce_process_bodies": (i32, [vp, vp, i32, vp, vp, vp, vp, i64, vp]),
        "pnce_draw_channel": (i32, [vp, i32, u64, vp, i64, vp]),
        "pnce_simulate_frames": (i32, [vp, vp, f64, u64, vp, i64, vp]),
        "pnce_kernel_launches": (i64, []),
    }
    for name, (res, args) in sig.items():
        if "PNCE_LIB" in os.environ and not hasattr(L, name):
            continue  # diagnostic override library (tools/bin) built from an older revision
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    """Raise the reference exception class matching a pnce_status_t."""
    if status == 0:
        return
    msg = lib().pnce_last_error().decode(errors="replace")
    raise _STATUS.get(status, E.DeviceError)(msg)
