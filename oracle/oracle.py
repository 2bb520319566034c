"""ctypes bindings for the CPU oracle (``sw_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline legs, never by the product package. Every
function mirrors a reference function (cited in ``sw_oracle.c``); the numpy
signatures follow ``swscan._compiled`` (src/_compiled.py:491-645) so the
parity tests read like the reference's own.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsworacle.so")
_lib = None

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

KERNEL_IDS = {"lazyf": 0, "lazyf-noexit": 1, "scan": 2}  # src/_compiled.py:576


def build() -> str:
    """Compile ``libsworacle.so`` with the committed Makefile."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "sw_oracle.c")
        ):
            build()
        L = C.CDLL(_LIB_PATH)
        L.swo_scan_steps.restype = C.c_int32
        L.swo_scan_steps.argtypes = [C.c_int64]
        L.swo_bias.restype = C.c_int64
        L.swo_bias.argtypes = [_i8p, C.c_int32]
        L.swo_build_profile.restype = C.c_int64
        L.swo_build_profile.argtypes = [_u8p, C.c_int64, _i8p, C.c_int32, C.c_int64, _u16p]
        L.swo_scalar.restype = C.c_int64
        L.swo_scalar.argtypes = [_u8p, C.c_int64, _u8p, C.c_int64, _i8p, C.c_int32, C.c_int64,
                                 C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.swo_align_lazyf.restype = C.c_int64
        L.swo_align_lazyf.argtypes = [_u16p, C.c_int64, C.c_int64, _u8p, C.c_int64, C.c_int64,
                                      C.c_int64, C.c_int64, C.c_int32, C.POINTER(C.c_uint8),
                                      _i64p, _i64p]
        L.swo_align_scan.restype = C.c_int64
        L.swo_align_scan.argtypes = [_u16p, C.c_int64, C.c_int64, _u8p, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_int64, C.POINTER(C.c_uint8), _i64p, _i64p]
        L.swo_scan_sequential.restype = None
        L.swo_scan_sequential.argtypes = [_u16p, C.c_int64, C.c_int64, _u16p]
        L.swo_weighted_max_scan.restype = None
        L.swo_weighted_max_scan.argtypes = [_u16p, C.c_int64, C.c_int64, _u16p]
        vp = C.c_void_p
        L.swo_batch_scalar.restype = None
        L.swo_batch_scalar.argtypes = [C.c_int64, _u8p, _i64p, _u8p, _i64p, vp, C.c_int32,
                                       C.c_int64, C.c_int64, vp, vp, vp, vp, _i64p, _i32p, _i32p,
                                       C.c_int32]
        L.swo_db_scalar.restype = None
        L.swo_db_scalar.argtypes = [_u8p, C.c_int64, C.c_int64, _u8p, _i64p, _i8p, C.c_int32,
                                    C.c_int64, C.c_int64, _i64p, _i32p, _i32p, C.c_int32]
        L.swo_batch_striped.restype = None
        L.swo_batch_striped.argtypes = [C.c_int32, C.c_int64, C.c_int64, _u8p, _i64p, _u8p, _i64p,
                                        vp, C.c_int32, C.c_int64, C.c_int64, vp, vp, vp, vp,
                                        _i64p, _u8p, _i64p, C.c_int32]
        L.swo_start_coords.restype = C.c_int32
        L.swo_start_coords.argtypes = [_u8p, _u8p, _i8p, C.c_int32, C.c_int64, C.c_int64,
                                       C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32)]
        L.swo_batch_starts.restype = None
        L.swo_batch_starts.argtypes = [C.c_int64, _u8p, _i64p, _u8p, _i64p, _i8p, C.c_int32,
                                       C.c_int64, C.c_int64, _i64p, _i32p, _i32p, _i32p, _i32p,
                                       C.c_int32]
        L.swo_db_striped.restype = None
        L.swo_db_striped.argtypes = [C.c_int32, _u16p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                     _u8p, _i64p, C.c_int64, C.c_int64, _i64p, _u8p, C.c_int32]
        _lib = L
    return _lib


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.uint8)


def _i8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.int8)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.int64)


def n_threads() -> int:
    return len(os.sched_getaffinity(0))


def bias_of(sub) -> int:
    sub = _i8(sub)
    return int(lib().swo_bias(sub.ravel(), sub.shape[0]))


def build_profile(query, sub, p: int) -> tuple[np.ndarray, int]:
    """Striped uint16 profile ``[A][L][p]`` + bias (``_build_profile_c``)."""
    q, s = _u8(query), _i8(sub)
    m = q.shape[0]
    L = (m + p - 1) // p
    prof = np.zeros((s.shape[0], L, p), dtype=np.uint16)
    bias = lib().swo_build_profile(q, m, s.ravel(), s.shape[0], p, prof.reshape(-1))
    return prof, int(bias)


def scalar(query, ref, sub, go: int, ge: int) -> tuple[int, int, int]:
    """Exact Gotoh score + first-max ``(ref_end, query_end)`` (``_sw_scalar_c`` + A10)."""
    q, r, s = _u8(query), _u8(ref), _i8(sub)
    ri, qi = C.c_int32(), C.c_int32()
    score = lib().swo_scalar(q, q.shape[0], r, r.shape[0], s.ravel(), s.shape[0], go, ge,
                             C.byref(ri), C.byref(qi))
    return int(score), int(ri.value), int(qi.value)


def align_prebuilt(kernel: str, prof: np.ndarray, bias: int, ref, go: int, ge: int):
    """``(score, overflow, counters[7], column_passes[n])`` as ``align_prebuilt``."""
    r = _u8(ref)
    prof = np.ascontiguousarray(prof, dtype=np.uint16)
    _, L, p = prof.shape
    sat = C.c_uint8()
    cnt = np.zeros(7, dtype=np.int64)
    colp = np.zeros(max(1, r.shape[0]), dtype=np.int64)
    kid = KERNEL_IDS[kernel]
    if kid == 2:
        score = lib().swo_align_scan(prof.reshape(-1), L, p, r, r.shape[0], bias, go, ge,
                                     C.byref(sat), cnt, colp)
    else:
        score = lib().swo_align_lazyf(prof.reshape(-1), L, p, r, r.shape[0], bias, go, ge,
                                      int(kid == 0), C.byref(sat), cnt, colp)
    return int(score), bool(sat.value), cnt, colp[: r.shape[0]]


def align_pair(kernel: str, p: int, query, ref, sub, go: int, ge: int):
    prof, bias = build_profile(query, sub, p)
    return align_prebuilt(kernel, prof, bias, ref, go, ge)


def weighted_max_scan(f, d: int) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.uint16)
    out = np.zeros_like(f)
    lib().swo_weighted_max_scan(f, f.shape[0], d, out)
    return out


def scan_sequential(f, d: int) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.uint16)
    out = np.zeros_like(f)
    lib().swo_scan_sequential(f, f.shape[0], d, out)
    return out


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def batch_scalar(flat_q, q_off, flat_r, r_off, sub=None, go=0, ge=0, match_a=None, mis_a=None,
                 go_a=None, ge_a=None, threads: int | None = None):
    """Pairwise oracle scores + coordinates (``batch_oracle_scores`` + A10)."""
    fq, qo, fr, ro = _u8(flat_q), _i64(q_off), _u8(flat_r), _i64(r_off)
    n = qo.shape[0] - 1
    score = np.zeros(n, dtype=np.int64)
    rend = np.zeros(n, dtype=np.int32)
    qend = np.zeros(n, dtype=np.int32)
    s = None if sub is None else _i8(sub)
    per = [None if x is None else _i64(x) for x in (match_a, mis_a, go_a, ge_a)]
    lib().swo_batch_scalar(n, fq, qo, fr, ro, _ptr(None if s is None else s.ravel()),
                           0 if s is None else s.shape[0], go, ge, *[_ptr(x) for x in per],
                           score, rend, qend, threads or n_threads())
    return score, rend, qend


def db_scalar(query, flat_r, r_off, sub, go: int, ge: int, threads: int | None = None):
    q, fr, ro, s = _u8(query), _u8(flat_r), _i64(r_off), _i8(sub)
    n = ro.shape[0] - 1
    score = np.zeros(n, dtype=np.int64)
    rend = np.zeros(n, dtype=np.int32)
    qend = np.zeros(n, dtype=np.int32)
    lib().swo_db_scalar(q, q.shape[0], n, fr, ro, s.ravel(), s.shape[0], go, ge, score, rend,
                        qend, threads or n_threads())
    return score, rend, qend


def batch_striped(kernel: str, p: int, flat_q, q_off, flat_r, r_off, sub=None, go=0, ge=0,
                  match_a=None, mis_a=None, go_a=None, ge_a=None, threads: int | None = None):
    """``batch_align`` (src/_compiled.py:504-529): scores, overflow, counters[n,7]."""
    fq, qo, fr, ro = _u8(flat_q), _i64(q_off), _u8(flat_r), _i64(r_off)
    n = qo.shape[0] - 1
    score = np.zeros(n, dtype=np.int64)
    over = np.zeros(n, dtype=np.uint8)
    cnt = np.zeros((n, 7), dtype=np.int64)
    s = None if sub is None else _i8(sub)
    per = [None if x is None else _i64(x) for x in (match_a, mis_a, go_a, ge_a)]
    lib().swo_batch_striped(KERNEL_IDS[kernel], p, n, fq, qo, fr, ro,
                            _ptr(None if s is None else s.ravel()),
                            0 if s is None else s.shape[0], go, ge, *[_ptr(x) for x in per],
                            score, over, cnt.reshape(-1), threads or n_threads())
    return score, over, cnt


def db_striped(kernel: str, prof: np.ndarray, bias: int, flat_r, r_off, go: int, ge: int,
               threads: int | None = None):
    prof = np.ascontiguousarray(prof, dtype=np.uint16)
    _, L, p = prof.shape
    fr, ro = _u8(flat_r), _i64(r_off)
    n = ro.shape[0] - 1
    score = np.zeros(n, dtype=np.int64)
    over = np.zeros(n, dtype=np.uint8)
    lib().swo_db_striped(KERNEL_IDS[kernel], prof.reshape(-1), L, p, bias, n, fr, ro, go, ge,
                         score, over, threads or n_threads())
    return score, over


def start_coords(query, ref, sub, go: int, ge: int, score: int, ref_end: int,
                 query_end: int) -> tuple[int, int]:
    """(ref_start, query_start) of the optimal alignment ending at the end cell
    (swo_start_coords); (-1, -1) for score 0."""
    rs, qs = C.c_int32(), C.c_int32()
    q, r = _u8(query), _u8(ref)
    if score > 0 and (ref_end >= r.shape[0] or query_end >= q.shape[0]):
        raise ValueError("end cell outside the sequences")
    rc = lib().swo_start_coords(q if q.size else np.zeros(1, np.uint8),
                                r if r.size else np.zeros(1, np.uint8), _i8(sub),
                                int(np.asarray(sub).shape[0]), go, ge, int(score), int(ref_end),
                                int(query_end), C.byref(rs), C.byref(qs))
    if rc != 0:
        raise ValueError("no alignment from the end cell reaches the score")
    return rs.value, qs.value


def batch_starts(flat_q, q_off, flat_r, r_off, sub, go: int, ge: int, score, ref_end, query_end,
                 threads: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    n = int(np.asarray(q_off).shape[0] - 1)
    rs = np.zeros(n, np.int32)
    qs = np.zeros(n, np.int32)
    fq, fr = _u8(flat_q), _u8(flat_r)
    lib().swo_batch_starts(n, fq if fq.size else np.zeros(1, np.uint8), _i64(q_off),
                           fr if fr.size else np.zeros(1, np.uint8), _i64(r_off), _i8(sub),
                           int(np.asarray(sub).shape[0]), go, ge, _i64(score),
                           np.ascontiguousarray(ref_end, dtype=np.int32),
                           np.ascontiguousarray(query_end, dtype=np.int32), rs, qs,
                           threads or n_threads())
    return rs, qs
