"""ctypes binding of the C ABI (include/monarch_b200.h).

The library is built in-tree (``paper_2602_12271_b200/libmonarch_b200.so``).
There is no fallback: if the library is missing or a call fails, this module
raises.  PyTorch supplies device memory and the current CUDA stream only.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MBX_LIB") or os.path.join(HERE, "libmonarch_b200.so")

ABI_VERSION = 1
F32, BF16 = 0, 1
FLAG_FORCE_GENERIC = 0x1
FLAG_NO_OUTPUT = 0x2
FLAG_FACTORS = 0x4
FLAG_NO_SPLIT = 0x8
FLAG_SPLIT = 0x10
FLAG_ALL_ITERS = 0x20

OK, BAD_SHAPE, BAD_PLAN, BAD_ITERS, BAD_EPS, BAD_DTYPE, NULL, WORKSPACE, UNSUPPORTED, CUDA = range(10)

EXPORTS = ("mbx_version", "mbx_last_error", "mbx_validate", "mbx_workspace_bytes",
           "mbx_selected_path", "mbx_forward", "mbx_apply", "mbx_apply_workspace_bytes",
           "mbx_profile_enable", "mbx_profile_collect", "mbx_profile_collect_ex", "mbx_token_index",
           "mbx_set_option", "mbx_backward", "mbx_backward_workspace_bytes")


class MbxDesc(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("batch", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("v_dim", ctypes.c_int32),
        ("c1_q", ctypes.c_int32),
        ("c1_kv", ctypes.c_int32),
        ("c2", ctypes.c_int32),
        ("s1", ctypes.c_int32),
        ("s2", ctypes.c_int32),
        ("iterations", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("eps_div", ctypes.c_double),
        ("eps_log", ctypes.c_double),
        ("q_stride", ctypes.c_int64 * 3),
        ("k_stride", ctypes.c_int64 * 3),
        ("v_stride", ctypes.c_int64 * 3),
        ("o_stride", ctypes.c_int64 * 3),
        ("q_order", ctypes.c_void_p),
        ("kv_order", ctypes.c_void_p),
        ("grid", ctypes.c_int32 * 3),
        ("nbhd", ctypes.c_int32 * 3),
    ]


class MbxError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"mbx status {status}: {message}")
        self.status = status


_lib = None


def load() -> ctypes.CDLL:
    """Load (never silently replace) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2602_12271_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    lib.mbx_version.restype = ctypes.c_int
    lib.mbx_last_error.restype = ctypes.c_char_p
    lib.mbx_validate.argtypes = [ctypes.POINTER(MbxDesc)]
    lib.mbx_validate.restype = ctypes.c_int
    lib.mbx_workspace_bytes.argtypes = [ctypes.POINTER(MbxDesc)]
    lib.mbx_workspace_bytes.restype = ctypes.c_size_t
    lib.mbx_apply_workspace_bytes.argtypes = [ctypes.POINTER(MbxDesc)]
    lib.mbx_apply_workspace_bytes.restype = ctypes.c_size_t
    lib.mbx_selected_path.argtypes = [ctypes.POINTER(MbxDesc)]
    lib.mbx_selected_path.restype = ctypes.c_int
    vp = ctypes.c_void_p
    lib.mbx_forward.argtypes = [ctypes.POINTER(MbxDesc), vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.mbx_forward.restype = ctypes.c_int
    lib.mbx_apply.argtypes = [ctypes.POINTER(MbxDesc), vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.mbx_apply.restype = ctypes.c_int
    lib.mbx_token_index.argtypes = [ctypes.POINTER(MbxDesc), ctypes.c_int, ctypes.c_int64]
    lib.mbx_token_index.restype = ctypes.c_int64
    lib.mbx_profile_enable.argtypes = [ctypes.c_int]
    lib.mbx_profile_enable.restype = ctypes.c_int
    lib.mbx_profile_collect.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_char_p),
                                        ctypes.c_int]
    lib.mbx_profile_collect.restype = ctypes.c_int
    lib.mbx_profile_collect_ex.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float),
                                           ctypes.POINTER(ctypes.c_char_p), ctypes.c_int]
    lib.mbx_profile_collect_ex.restype = ctypes.c_int
    lib.mbx_backward.argtypes = [ctypes.POINTER(MbxDesc), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t,
                                 vp]
    lib.mbx_backward.restype = ctypes.c_int
    lib.mbx_backward_workspace_bytes.argtypes = [ctypes.POINTER(MbxDesc)]
    lib.mbx_backward_workspace_bytes.restype = ctypes.c_size_t
    lib.mbx_set_option.argtypes = [ctypes.c_char_p, ctypes.c_int]
    lib.mbx_set_option.restype = ctypes.c_int
    if lib.mbx_version() != ABI_VERSION:
        raise ImportError(f"libmonarch_b200 ABI {lib.mbx_version()} != {ABI_VERSION}; rebuild")
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != OK:
        raise MbxError(status, load().mbx_last_error().decode())


def profile_collect(max_entries: int = 4096) -> list[tuple[str, float]]:
    """Per-launch (kernel name, ms) recorded since profiling was enabled."""
    return [(n, ms) for n, _, ms in profile_collect_ex(max_entries)]


def profile_collect_ex(max_entries: int = 4096) -> list[tuple[str, float, float]]:
    """Per-launch (kernel name, start ms relative to the first launch, ms)."""
    lib = load()
    st = (ctypes.c_float * max_entries)()
    ms = (ctypes.c_float * max_entries)()
    names = (ctypes.c_char_p * max_entries)()
    n = lib.mbx_profile_collect_ex(st, ms, names, max_entries)
    return [(names[i].decode(), float(st[i]), float(ms[i])) for i in range(min(n, max_entries))]


# bumped on every option change: options such as MBX_WAVE / MBX_WS_CAP_MB change the
# workspace size, so host-side caches of mbx_workspace_bytes key on it
OPTIONS_VERSION = [0]


def set_option(name: str, value: int) -> int:
    """Process-wide diagnostic option (mbx_set_option); returns the previous value."""
    prev = load().mbx_set_option(name.encode(), int(value))
    if prev == -1000:
        raise KeyError(name)
    OPTIONS_VERSION[0] += 1
    return prev
