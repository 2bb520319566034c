"""ctypes binding of libswscan_b200.so (the C ABI declared in include/swscan_b200.h).

The product path has no CPU fallback: if the shared library is missing or the
process has no CUDA device, every entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SWB_LIB_PATH") or os.path.join(PKG_DIR, "libswscan_b200.so")
CSRC = os.path.join(PKG_DIR, "csrc")

SW_OK, SW_EINVAL, SW_ECUDA, SW_ENOTSUP = 0, -1, -2, -3
KERNEL_IDS = {  # reference _KERNEL_IDS (src/_compiled.py:576) + parity-mode lazy-F
    "lazyf": 0,
    "lazyf-noexit": 1,
    "scan": 2,
    "lazyf-mirror": 3,
    "lazyf-noexit-mirror": 4,
    "wavefront": 5,  # sw_align_long only: strip pipeline with an intra-strip wavefront
}
FLAG_REF_OVERFLOW, FLAG_RESCUE, FLAG_RESCUED, FLAG_FEED_TIMEOUT = 1, 2, 4, 8

EXPORTS = (
    "sw_version",
    "sw_last_error",
    "sw_plan_query",
    "sw_profile_build",
    "sw_db_align",
    "sw_pairs_align",
    "sw_collect_flagged",
    "sw_topk_workspace",
    "sw_topk",
    "sw_unpack_2bit",
    "sw_scan_lanes",
    "sw_dpx_probe",
    "sw_long_workspace_bytes",
    "sw_align_long",
    "sw_block_plan",
    "sw_align_block",
)


class NativeUnavailable(RuntimeError):
    """The CUDA library could not be loaded; there is deliberately no fallback."""


class SwError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libswscan_b200 error {code}: {msg}")
        self.code = code


class DbOpts(C.Structure):
    """sw_db_opts_t (include/swscan_b200.h): coordinate floor + streamed-input feed."""

    _fields_ = [
        ("d_coord_floor", C.c_void_p),
        ("floor_sample", C.c_int64),
        ("floor_k", C.c_int32),
        ("arrive_epoch", C.c_int32),
        ("d_arrived", C.c_void_p),
        ("arrive_jobs", C.c_int64),
        ("arrive_timeout_ns", C.c_int64),
    ]


class Plan(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("lanes", C.c_int32),
        ("threads", C.c_int32),
        ("seg_len", C.c_int32),
        ("lmax", C.c_int32),
        ("m", C.c_int32),
        ("n_sym", C.c_int32),
        ("prof_words", C.c_int32),
    ]

    def __repr__(self) -> str:
        return ("Plan(" + ", ".join(f"{k}={getattr(self, k)}" for k, _ in self._fields_) + ")")


_lib = None


def build(force: bool = False) -> str:
    """Compile the CUDA library in-tree with the committed Makefile (nvcc, sm_100a)."""
    if force or not os.path.exists(LIB_PATH) or _stale():
        jobs = str(max(1, min(16, os.cpu_count() or 1)))
        subprocess.run(["make", "-s", "-j", jobs, "-C", CSRC], check=True)
    return LIB_PATH


def _stale() -> bool:
    t = os.path.getmtime(LIB_PATH)
    for root in (CSRC, os.path.join(os.path.dirname(PKG_DIR), "include")):
        for f in os.listdir(root):
            if f.endswith((".cu", ".cuh", ".inc", ".h")) and os.path.getmtime(os.path.join(root, f)) > t:
                return True
    return False


def load():
    """Load the library (no CUDA context is created here)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(f"{LIB_PATH} not built; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.sw_version.restype = i32
    L.sw_version.argtypes = []
    L.sw_last_error.restype = C.c_char_p
    L.sw_last_error.argtypes = []
    L.sw_plan_query.restype = i32
    L.sw_plan_query.argtypes = [i32, i32, i32, i32, C.POINTER(Plan)]
    L.sw_profile_build.restype = i32
    L.sw_profile_build.argtypes = [C.POINTER(Plan), vp, vp, i32, vp, vp]
    L.sw_db_align.restype = i32
    L.sw_db_align.argtypes = [C.POINTER(Plan), vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, i64,
                              vp, vp, vp, vp, vp, vp, vp, C.POINTER(DbOpts), vp]
    L.sw_pairs_align.restype = i32
    L.sw_pairs_align.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, i64, vp, i32, i32, vp, i32,
                                 i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.sw_collect_flagged.restype = i32
    L.sw_collect_flagged.argtypes = [vp, i64, C.c_uint8, vp, vp, vp]
    L.sw_topk_workspace.restype = i64
    L.sw_topk_workspace.argtypes = []
    L.sw_topk.restype = i32
    L.sw_topk.argtypes = [vp, vp, vp, vp, i64, i32, vp, vp, vp]
    L.sw_unpack_2bit.restype = i32
    L.sw_unpack_2bit.argtypes = [vp, i64, vp, vp]
    L.sw_scan_lanes.restype = i32
    L.sw_scan_lanes.argtypes = [i32, i32, vp, vp, i32, vp, vp]
    L.sw_dpx_probe.restype = i64
    L.sw_dpx_probe.argtypes = [i32, i64, vp, vp]
    L.sw_long_workspace_bytes.restype = i64
    L.sw_long_workspace_bytes.argtypes = [i64, i64, i32, i32]
    L.sw_align_long.restype = i32
    L.sw_align_long.argtypes = [i32, i32, vp, i64, vp, i64, vp, i32, i32, i32, i32, i32, vp, i64,
                                vp, vp, vp, vp, vp]
    L.sw_block_plan.restype = i32
    L.sw_block_plan.argtypes = [i32, i32, i64, i32, i32, C.POINTER(C.c_int32)]
    L.sw_align_block.restype = i32
    L.sw_align_block.argtypes = [i32, i32, i32, vp, i64, vp, i64, vp, i32, i32, i32, i32, i32, i32,
                                 vp, vp, vp, vp, vp, vp, vp]
    _lib = _Strict(L)
    return _lib


class _Strict:
    """The loaded library with arity-checked entry points: ctypes passes surplus
    arguments of a function with argtypes through as varargs, which for this C ABI
    would silently shift the stream argument; here a wrong argument count raises."""

    def __init__(self, lib):
        self._lib = lib
        for name in EXPORTS:
            fn = getattr(lib, name)
            setattr(self, name, self._wrap(name, fn))

    @staticmethod
    def _wrap(name, fn):
        n = len(fn.argtypes)

        def call(*args):
            if len(args) != n:
                raise TypeError(f"{name}() takes {n} arguments ({len(args)} given)")
            return fn(*args)

        call.__name__ = name
        return call

    def __getattr__(self, name):
        return getattr(self._lib, name)


def check(rc: int) -> None:
    if rc != SW_OK:
        raise SwError(rc, load().sw_last_error().decode(errors="replace"))


def plan_query(m: int, n_sym: int, width: int, lanes: int = 0) -> Plan:
    p = Plan()
    check(load().sw_plan_query(int(m), int(n_sym), int(width), int(lanes), C.byref(p)))
    return p


def block_plan(m: int, n_sym: int, width: int = 16, kernel: int = 2, lanes: int = 0):
    """Layout of the block / cluster kernel: (lanes, threads per CTA, CTAs per cluster,
    seg_len), or None when no layout exists (sw_block_plan)."""
    out = (C.c_int32 * 4)()
    rc = load().sw_block_plan(int(width), int(kernel), int(m), int(n_sym), int(lanes), out)
    if rc == SW_ENOTSUP:
        return None
    check(rc)
    return tuple(int(x) for x in out)
