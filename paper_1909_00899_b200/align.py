"""Reference-compatible alignment entry points on the B200 kernels.

Mirrors the reference operator interface (``swscan._compiled`` and the pure
kernels): ``build_profile_arrays`` / ``align_prebuilt`` / ``align_pair`` /
``scalar_score`` / ``batch_align`` / ``batch_oracle_scores`` keep their names,
argument meaning and error behaviour (src/_compiled.py:491-645,
src/kernels.py:62-264). Differences, all documented in DESIGN.md:

* results carry exact end coordinates ``ref_end`` / ``query_end``;
* ``score`` is always exact: 16-bit runs that approach the wrap guard are
  re-run in 32 bits on the device; ``overflow`` keeps the reference meaning
  (the uint16 reference kernels would saturate, i.e. exact > 65535 - bias);
* ``p`` selects the reference stripe count when a compiled kernel instance
  exists for it, otherwise the throughput layout is used (scores and end
  coordinates do not depend on p; per-column pass counts do).

Device memory and streams come from torch; the compute is the CUDA library
(``_lib``). There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .scoring import ScoringScheme, SymbolOutOfAlphabet


class ProfileMismatch(ValueError):
    """Profile was built for a different scheme or vector shape (src/kernels.py:27-28)."""


class EmptyQuery(ValueError):
    """Profile construction requires at least one query residue (src/profile.py:18-19)."""


@dataclass
class OpCounters:
    """Reference vector-op tally (src/vectors.py:61-95), reconstructed in closed
    form from the device's per-column pass counts."""

    shifts: int = 0
    sat_adds: int = 0
    sat_subs: int = 0
    maxes: int = 0
    loads: int = 0
    stores: int = 0
    correction_passes: int = 0

    @property
    def vec_ops_total(self) -> int:
        return self.shifts + self.sat_adds + self.sat_subs + self.maxes + self.loads + self.stores


@dataclass
class AlignmentResult:
    """src/kernels.py:62-76 plus end coordinates (0-based, -1 when score is 0)."""

    score: int
    overflow: bool
    counters: OpCounters | None
    correction_passes: int
    column_passes: tuple[int, ...]
    ref_end: int = -1
    query_end: int = -1
    lanes: int = 0
    seg_len: int = 0
    rescued: bool = False


def scan_steps(p: int) -> int:
    """_scan_steps, src/_compiled.py:39-46."""
    s = 0
    while (1 << s) < p:
        s += 1
    return max(1, s)


def counters_from_passes(kernel: str, n: int, L: int, p: int, passes: np.ndarray) -> OpCounters:
    """Closed-form reference counters (src/_compiled.py:137-219, :246-339)."""
    if kernel == "scan":
        s = scan_steps(p)
        return OpCounters(shifts=n * (2 + s), sat_adds=n * L, sat_subs=n * (1 + 5 * L + s),
                          maxes=n * (1 + 6 * L + s), loads=n * (1 + 3 * L), stores=n * 2 * L,
                          correction_passes=n * s)
    k = int(passes.sum())
    early = kernel.startswith("lazyf") and "noexit" not in kernel
    broke = int(np.count_nonzero(passes < p)) if early else 0
    return OpCounters(shifts=n + k + broke, sat_adds=n * L, sat_subs=n * 4 * L + k * L,
                      maxes=n * 5 * L + k * L, loads=n * (1 + 3 * L) + k * L,
                      stores=n * 2 * L + k * L, correction_passes=k)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _to_dev(x, dtype: torch.dtype) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x))).to(device="cuda", dtype=dtype)


def _require_cuda() -> None:
    _lib.load()
    if not torch.cuda.is_available():
        raise _lib.NativeUnavailable("no CUDA device: the B200 kernels have no CPU fallback")


def _codes(seq, n_sym: int, what: str) -> np.ndarray:
    if isinstance(seq, torch.Tensor):
        arr = seq.detach().cpu().numpy()
    else:
        arr = np.asarray(seq)
    arr = arr.astype(np.int64, copy=False).ravel()
    if arr.size and (arr.min() < 0 or arr.max() >= n_sym):
        bad = int(arr[(arr < 0) | (arr >= n_sym)][0])
        raise SymbolOutOfAlphabet(f"{what} index {bad} outside 0..{n_sym - 1}")
    return arr.astype(np.uint8)


def _kernel_id(kernel: str) -> int:
    return _lib.KERNEL_IDS[kernel]  # KeyError on unknown names, as the reference


@dataclass
class DeviceProfile:
    """Striped query profile resident in HBM (reference: the (prof, bias) pair of
    build_profile_arrays, src/_compiled.py:579-585), 16-bit layout plus the
    32-bit layout used by overflow rescues."""

    scheme: ScoringScheme
    m: int
    query: torch.Tensor
    sub: torch.Tensor
    bias: int
    max_sub: int
    plan16: _lib.Plan
    prof16: torch.Tensor
    requested_lanes: int = 0
    plan32: _lib.Plan | None = None
    prof32: torch.Tensor | None = None
    long32: bool = False  # no 32-bit warp-kernel plan: rescues use the strip pipeline
    extra: dict = field(default_factory=dict)

    # The reference returns a (prof, bias) tuple and its callers unpack it
    # (`prof, bias = build_profile_arrays(...)`, src/runner.py:146,
    # src/_compiled.py:614): a DeviceProfile unpacks as (itself, bias), so
    # align_prebuilt(kernel, prof, bias, ref, scheme) works unchanged.
    def __iter__(self):
        return iter((self, self.bias))

    def __len__(self) -> int:
        return 2

    def __getitem__(self, i: int):
        return (self, self.bias)[i]

    @property
    def seg_len(self) -> int:
        return self.plan16.seg_len

    @property
    def lanes(self) -> int:
        return self.plan16.lanes

    def for_kernel(self, kernel: str) -> tuple[_lib.Plan, torch.Tensor]:
        """16-bit (plan, profile) usable by `kernel`: segments beyond 32 words exist
        only for the scan kernel, so other kernels get a <= 32-word layout."""
        if kernel == "scan" or self.plan16.lmax <= 32:
            return self.plan16, self.prof16
        if "short" not in self.extra:
            P = 8
            while (self.m + P - 1) // P > 32:
                P *= 2
            plan = _lib.plan_query(self.m, self.scheme.n_symbols, 16, P)
            prof = torch.empty(plan.prof_words, dtype=torch.int32, device="cuda")
            _lib.check(_lib.load().sw_profile_build(C.byref(plan), _ptr(self.query), _ptr(self.sub),
                                                     self.bias, _ptr(prof), _stream()))
            self.extra["short"] = (plan, prof)
        return self.extra["short"]

    def ensure32(self) -> None:
        """Build the 32-bit profile used by overflow rescues. A query longer than the
        32-bit warp kernels hold (1,024 residues) has none: its rare rescues run
        through the 32-bit strip pipeline instead (rescue_long)."""
        if self.plan32 is not None or self.long32:
            return
        lanes = self.requested_lanes if self.requested_lanes and self.requested_lanes <= 32 else 0
        try:
            self.plan32 = _lib.plan_query(self.m, self.scheme.n_symbols, 32, lanes)
        except _lib.SwError:
            try:
                self.plan32 = _lib.plan_query(self.m, self.scheme.n_symbols, 32, 0)
            except _lib.SwError:
                self.long32 = True
                return
        self.prof32 = torch.empty(self.plan32.prof_words, dtype=torch.int32, device="cuda")
        _lib.check(_lib.load().sw_profile_build(C.byref(self.plan32), _ptr(self.query),
                                                 _ptr(self.sub), self.bias, _ptr(self.prof32),
                                                 _stream()))


def _plan_with_fallback(m: int, n_sym: int, width: int, lanes: int) -> _lib.Plan:
    if lanes:
        try:
            return _lib.plan_query(m, n_sym, width, lanes)
        except _lib.SwError:
            pass
    return _lib.plan_query(m, n_sym, width, 0)


def as_scheme(scheme) -> ScoringScheme:
    """Accept the reference's own ScoringScheme (src/scoring.py:56-98) or any object
    with its fields (matrix, gap_open, gap_extend), so reference callers can pass
    theirs unchanged; validation is the reference's (ValueError)."""
    if isinstance(scheme, ScoringScheme):
        return scheme
    return ScoringScheme(scheme.matrix, scheme.gap_open, scheme.gap_extend)


def build_profile_arrays(query, scheme: ScoringScheme, p: int = 0) -> DeviceProfile:
    """Build the striped profile on the device (src/_compiled.py:579-585).
    Unpacks as ``(prof, bias)`` like the reference's tuple."""
    _require_cuda()
    scheme = as_scheme(scheme)
    q = _codes(query, scheme.n_symbols, "query")
    if q.size == 0:
        raise EmptyQuery("query must contain at least one residue")
    qd = torch.from_numpy(q).cuda()
    sub = torch.from_numpy(scheme.as_array()).cuda()
    try:
        plan = _plan_with_fallback(int(q.size), scheme.n_symbols, 16, int(p))
    except _lib.SwError:
        # longer than the warp kernels hold: the strip pipeline (align_long) runs it
        return DeviceProfile(scheme, int(q.size), qd, sub, scheme.bias, scheme.max_score, None,
                             None, requested_lanes=int(p))
    prof = torch.empty(plan.prof_words, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().sw_profile_build(C.byref(plan), _ptr(qd), _ptr(sub), scheme.bias,
                                             _ptr(prof), _stream()))
    return DeviceProfile(scheme, int(q.size), qd, sub, scheme.bias, scheme.max_score, plan, prof,
                         requested_lanes=int(p))


def align_long(query, ref, scheme: ScoringScheme, width: int = 32, kernel: str = "scan",
               query_dev: torch.Tensor | None = None, ref_dev: torch.Tensor | None = None,
               coords: bool = True) -> dict:
    """One long pair through the strip pipeline (sw_align_long). Returns host ints
    ``score, ref_end, query_end, flags``; a 16-bit run that hits the wrap guard is
    repeated in 32 bits. ``coords=False``: score-only launch (ends stay -1)."""
    _require_cuda()
    L = _lib.load()
    qd = query_dev if query_dev is not None else torch.from_numpy(
        _codes(query, scheme.n_symbols, "query")).cuda()
    rd = ref_dev if ref_dev is not None else torch.from_numpy(
        _codes(ref, scheme.n_symbols, "reference")).cuda()
    m, n = int(qd.numel()), int(rd.numel())
    if m == 0 or n == 0:
        return {"score": 0, "ref_end": -1, "query_end": -1, "flags": 0}
    sub = torch.from_numpy(scheme.as_array()).cuda()
    out = torch.zeros(4, dtype=torch.int32, device="cuda")
    fl = torch.zeros(1, dtype=torch.uint8, device="cuda")
    for w in ((16, 32) if width == 16 and kernel != "wavefront" else (32,)):
        nbytes = L.sw_long_workspace_bytes(m, n, scheme.n_symbols, w)
        if nbytes < 0:
            _lib.check(int(nbytes))
        ws = torch.empty(int(nbytes), dtype=torch.uint8, device="cuda")
        _lib.check(L.sw_align_long(w, _kernel_id(kernel), _ptr(qd), m, _ptr(rd), n, _ptr(sub),
                                   scheme.n_symbols, scheme.gap_open, scheme.gap_extend,
                                   scheme.bias, scheme.max_score, _ptr(ws), int(nbytes),
                                   C.c_void_p(out.data_ptr()),
                                   C.c_void_p(out.data_ptr() + 4) if coords else None,
                                   C.c_void_p(out.data_ptr() + 8) if coords else None,
                                   _ptr(fl), _stream()))
        flags = int(fl.item())
        if not flags & _lib.FLAG_RESCUE:
            break
    o = out.cpu().tolist()
    if not coords:
        o[1] = o[2] = -1
    if width == 16 and w == 32:
        flags |= _lib.FLAG_RESCUED
    return {"score": o[0], "ref_end": o[1], "query_end": o[2], "flags": flags & ~_lib.FLAG_RESCUE}


def align_block(query, ref, scheme: ScoringScheme, p: int = 0, kernel: str = "scan",
                width: int = 16, coords: bool = True, col_passes: bool = False,
                query_dev: torch.Tensor | None = None, ref_dev: torch.Tensor | None = None) -> dict:
    """One pair on the block / cluster kernel (sw_align_block): the reference layout
    VectorSpec(p) for p beyond one warp, the F scan resolved warp -> block -> cluster
    (DSMEM). ``p = 0`` chooses the layout. Returns host values ``score, ref_end,
    query_end, flags, lanes, threads, cluster, seg_len`` (+ ``col_passes``,
    ``pass_stats`` for lazy-F); a 16-bit run that hits the wrap guard is repeated in
    32 bits."""
    _require_cuda()
    L = _lib.load()
    kid = _kernel_id(kernel)
    if kid == _lib.KERNEL_IDS["wavefront"]:
        raise _lib.SwError(_lib.SW_ENOTSUP, "the block kernel runs scan and lazy-F")
    qd = query_dev if query_dev is not None else torch.from_numpy(
        _codes(query, scheme.n_symbols, "query")).cuda()
    rd = ref_dev if ref_dev is not None else torch.from_numpy(
        _codes(ref, scheme.n_symbols, "reference")).cuda()
    m, n = int(qd.numel()), int(rd.numel())
    if m == 0 or n == 0:
        return {"score": 0, "ref_end": -1, "query_end": -1, "flags": 0}
    sub = torch.from_numpy(scheme.as_array()).cuda()
    out = torch.zeros(4, dtype=torch.int32, device="cuda")
    fl = torch.zeros(1, dtype=torch.uint8, device="cuda")
    passes = torch.zeros(n, dtype=torch.int32, device="cuda") if col_passes else None
    stats = torch.zeros(2, dtype=torch.int64, device="cuda") if kernel != "scan" else None
    res = {}
    for w in ((16, 32) if width == 16 else (32,)):
        geo = _lib.block_plan(m, scheme.n_symbols, w, kid, p)
        if geo is None:
            if w == 32 and width == 16:
                geo = _lib.block_plan(m, scheme.n_symbols, 32, kid, 0)  # rescue at any layout
            if geo is None:
                raise _lib.SwError(_lib.SW_ENOTSUP, f"no block layout for m={m}, p={p}, width={w}")
        _lib.check(L.sw_align_block(w, kid, geo[0], _ptr(qd), m, _ptr(rd), n, _ptr(sub),
                                    scheme.n_symbols, scheme.gap_open, scheme.gap_extend,
                                    scheme.bias, scheme.max_score, int(bool(coords)),
                                    C.c_void_p(out.data_ptr()), C.c_void_p(out.data_ptr() + 4),
                                    C.c_void_p(out.data_ptr() + 8), _ptr(fl), _ptr(passes),
                                    _ptr(stats), _stream()))
        flags = int(fl.item())
        res = {"lanes": geo[0], "threads": geo[1], "cluster": geo[2], "seg_len": geo[3]}
        if not flags & _lib.FLAG_RESCUE:
            break
    o = out.cpu().tolist()
    if not coords:
        o[1] = o[2] = -1
    if width == 16 and w == 32:
        flags |= _lib.FLAG_RESCUED
    res.update(score=o[0], ref_end=o[1], query_end=o[2], flags=flags & ~_lib.FLAG_RESCUE)
    if passes is not None:
        res["col_passes"] = passes.cpu().numpy()
    if stats is not None:
        res["pass_stats"] = tuple(int(x) for x in stats.cpu().tolist())
    return res


def db_align(prof: DeviceProfile, tgt: torch.Tensor, start: torch.Tensor, length: torch.Tensor,
             order: torch.Tensor | None = None, kernel: str = "scan",
             col_passes: torch.Tensor | None = None, out: dict | None = None,
             rescue: bool = True, coord_floor: torch.Tensor | None = None) -> dict:
    """All-device database alignment: one profile vs n targets, 16-bit with a
    device-side 32-bit rescue of wrap-guard hits. Returns dict of device tensors
    ``score, ref_end, query_end, flags`` indexed by target id. ``coord_floor``
    (device int32 [1]): locate end coordinates only for scores >= the floor."""
    L = _lib.load()
    n = int(length.shape[0])
    if out is None:
        out = {
            "score": torch.empty(n, dtype=torch.int32, device="cuda"),
            "ref_end": torch.empty(n, dtype=torch.int32, device="cuda"),
            "query_end": torch.empty(n, dtype=torch.int32, device="cuda"),
            "flags": torch.empty(n, dtype=torch.uint8, device="cuda"),
        }
    kid = _kernel_id(kernel)
    sch = prof.scheme
    st = _stream()
    plan16, prof16 = prof.for_kernel(kernel)
    _lib.check(L.sw_db_align(C.byref(plan16), _ptr(prof16), kid, sch.gap_open,
                             sch.gap_extend, prof.bias, prof.max_sub, _ptr(tgt), _ptr(start),
                             _ptr(length), _ptr(order), n, None, _ptr(out["score"]),
                             _ptr(out["ref_end"]), _ptr(out["query_end"]), _ptr(out["flags"]),
                             _ptr(col_passes), None, (C.byref(_lib.DbOpts(d_coord_floor=coord_floor.data_ptr())) if coord_floor is not None else None), st))
    if rescue:
        _rescue_db(prof, tgt, start, length, kid, col_passes, out, n)
    return out


def _rescue_db(prof, tgt, start, length, kid, col_passes, out, n) -> None:
    L = _lib.load()
    ws = out.get("_rescue")
    if ws is None or ws[0].shape[0] < n:
        ws = (torch.empty(max(n, 1), dtype=torch.int32, device="cuda"),
              torch.zeros(1, dtype=torch.int64, device="cuda"))
        out["_rescue"] = ws
    st = _stream()
    prof.ensure32()
    if prof.long32:
        rescue_long(prof, tgt, start, length, out, n)
        return
    _lib.check(L.sw_collect_flagged(_ptr(out["flags"]), n, _lib.FLAG_RESCUE, _ptr(ws[0]),
                                    _ptr(ws[1]), st))
    sch = prof.scheme
    _lib.check(L.sw_db_align(C.byref(prof.plan32), _ptr(prof.prof32), kid, sch.gap_open,
                             sch.gap_extend, prof.bias, prof.max_sub, _ptr(tgt), _ptr(start),
                             _ptr(length), _ptr(ws[0]), 0, _ptr(ws[1]), _ptr(out["score"]),
                             _ptr(out["ref_end"]), _ptr(out["query_end"]), _ptr(out["flags"]),
                             _ptr(col_passes), None, None, st))


def rescue_long(prof, tgt, start, length, out, n) -> None:
    """Exact 32-bit re-run of the 16-bit wrap-guard hits of a query too long for the
    32-bit warp kernels: each flagged target goes through the 32-bit scan strip
    pipeline (sw_align_long). Reads the flags on the host (these are rare: the
    alignment score must approach 32,767)."""
    fl = out["flags"][:n]
    hits = torch.nonzero((fl & _lib.FLAG_RESCUE) != 0).flatten().tolist()
    for j in hits:
        s0, ln = int(start[j]), int(length[j])
        r = align_long(None, None, prof.scheme, width=32, query_dev=prof.query,
                       ref_dev=tgt[s0:s0 + ln])
        out["score"][j] = r["score"]
        out["ref_end"][j] = r["ref_end"]
        out["query_end"][j] = r["query_end"]
        out["flags"][j] = (r["flags"] & _lib.FLAG_REF_OVERFLOW) | _lib.FLAG_RESCUED


def _result_from(prof_or_none, kernel, n, L_, P, score, flags, rend, qend, passes) -> AlignmentResult:
    fl = int(flags)
    passes_np = np.asarray(passes, dtype=np.int64) if passes is not None else np.zeros(n, np.int64)
    if P == 0:  # strip pipeline: no single reference layout to reconstruct counters for
        return AlignmentResult(score=int(score), overflow=bool(fl & _lib.FLAG_REF_OVERFLOW),
                               counters=None, correction_passes=0, column_passes=(),
                               ref_end=int(rend), query_end=int(qend),
                               rescued=bool(fl & _lib.FLAG_RESCUED))
    if kernel == "scan":
        passes_np = np.full(n, scan_steps(P), dtype=np.int64)
    cnt = counters_from_passes(kernel, n, L_, P, passes_np) if n > 0 else OpCounters()
    return AlignmentResult(score=int(score), overflow=bool(fl & _lib.FLAG_REF_OVERFLOW),
                           counters=cnt, correction_passes=cnt.correction_passes,
                           column_passes=tuple(int(x) for x in passes_np), ref_end=int(rend),
                           query_end=int(qend), lanes=P, seg_len=L_,
                           rescued=bool(fl & _lib.FLAG_RESCUED))


def align_prebuilt(kernel: str, prof: DeviceProfile, bias=None, ref=None,
                   scheme: ScoringScheme | None = None) -> AlignmentResult:
    """One alignment against a prebuilt device profile (src/_compiled.py:588-607)."""
    if not isinstance(prof, DeviceProfile):
        raise ProfileMismatch("align_prebuilt needs a DeviceProfile from build_profile_arrays")
    if scheme is not None and (scheme.matrix != prof.scheme.matrix
                               or scheme.gap_open != prof.scheme.gap_open
                               or scheme.gap_extend != prof.scheme.gap_extend):
        raise ProfileMismatch("profile was built for a different scoring scheme")
    if bias is not None and int(bias) != prof.bias:
        raise ProfileMismatch("profile was built for a different scoring scheme")
    kid = _kernel_id(kernel)
    r = _codes(ref, prof.scheme.n_symbols, "reference")
    n = int(r.size)
    if n == 0:
        return _result_from(None, kernel, 0, prof.seg_len if prof.plan16 else 0,
                            prof.lanes if prof.plan16 else 0, 0, 0, -1, -1, None)
    if prof.requested_lanes > 64 and _lib.block_plan(prof.m, prof.scheme.n_symbols, 16, kid,
                                                     prof.requested_lanes) is not None:
        # the reference layout VectorSpec(p) beyond one warp: block / cluster kernel
        o = align_block(None, r, prof.scheme, prof.requested_lanes, kernel, 16,
                        col_passes=kernel != "scan", query_dev=prof.query)
        return _result_from(prof, kernel, n, o["seg_len"], o["lanes"], o["score"], o["flags"],
                            o["ref_end"], o["query_end"], o.get("col_passes"))
    long_query = prof.plan16 is None
    if not long_query and prof.plan32 is None:
        prof.ensure32()
        if prof.long32:
            long_query = None  # 16-bit warp kernel; a rescue needs the strip pipeline
    if long_query:
        if kernel != "scan":
            raise _lib.SwError(_lib.SW_ENOTSUP,
                               f"query of {prof.m} residues: only the scan kernel runs as a strip pipeline")
        o = align_long(None, r, prof.scheme, 16, kernel, query_dev=prof.query)
        return _result_from(None, kernel, n, 0, 0, o["score"], o["flags"], o["ref_end"],
                            o["query_end"], None)
    tgt = torch.from_numpy(r).cuda()
    start = torch.zeros(1, dtype=torch.int64, device="cuda")
    length = torch.full((1,), n, dtype=torch.int32, device="cuda")
    passes = torch.zeros(n, dtype=torch.int32, device="cuda") if kid != 2 else None
    if long_query is None:
        out = db_align(prof, tgt, start, length, None, kernel, passes, rescue=False)
        if int(out["flags"][0]) & _lib.FLAG_RESCUE:
            o = align_long(None, None, prof.scheme, 32, "scan", query_dev=prof.query, ref_dev=tgt)
            return _result_from(None, kernel, n, 0, 0, o["score"], o["flags"] | _lib.FLAG_RESCUED,
                                o["ref_end"], o["query_end"], None)
    else:
        out = db_align(prof, tgt, start, length, None, kernel, passes)
    flags = int(out["flags"][0])
    if flags & _lib.FLAG_RESCUED:
        P, L_ = (prof.plan32.lanes, prof.plan32.seg_len) if prof.plan32 is not None else (0, 0)
    else:
        pl = prof.for_kernel(kernel)[0]
        P, L_ = pl.lanes, pl.seg_len
    return _result_from(prof, kernel, n, L_, P, int(out["score"][0]), flags,
                        int(out["ref_end"][0]), int(out["query_end"][0]),
                        passes.cpu().numpy() if passes is not None else None)


def align_pair(kernel: str, p: int, query, ref, scheme: ScoringScheme) -> AlignmentResult:
    """src/_compiled.py:610-615."""
    return align_prebuilt(kernel, build_profile_arrays(query, scheme, p), ref=ref, scheme=scheme)


def scalar_score(query, ref, scheme: ScoringScheme) -> int:
    """Exact local score (src/_compiled.py:618-625), computed by the device kernel."""
    q = _codes(query, scheme.n_symbols, "query")
    r = _codes(ref, scheme.n_symbols, "reference")
    if q.size == 0 or r.size == 0:
        return 0
    return align_pair("scan", 0, q, r, scheme).score


def counters_from_stats(kernel: str, n: int, L: int, p: int, total_passes: int,
                        breaks: int) -> list[int]:
    """Reference op counters (src/_compiled.py:137-219, :246-339) of one alignment
    from its column count n, layout (L, p) and device pass statistics."""
    if n <= 0:
        return [0] * 7
    if kernel == "scan":
        c = counters_from_passes("scan", n, L, p, np.zeros(0))
    else:
        k = int(total_passes)
        c = OpCounters(shifts=n + k + int(breaks), sat_adds=n * L, sat_subs=n * 4 * L + k * L,
                       maxes=n * 5 * L + k * L, loads=n * (1 + 3 * L) + k * L,
                       stores=n * 2 * L + k * L, correction_passes=k)
    return [c.shifts, c.sat_adds, c.sat_subs, c.maxes, c.loads, c.stores, c.correction_passes]


def pairs_align(flat_q, q_off, flat_r, r_off, *, kernel: str = "scan", lanes: int = 0,
                scheme: ScoringScheme | None = None, match_a=None, mis_a=None, go_a=None,
                ge_a=None, width: int = 16, stats: bool = False, coords: bool = True) -> dict:
    """Independent pairs (CSR queries/targets), results as numpy arrays
    ``score, ref_end, query_end, flags`` (+ ``pass_stats``, ``lanes_used``,
    ``seg_len`` with ``stats=True``). ``coords=False``: score-only launches (no
    end-coordinate search; ``ref_end``/``query_end`` stay -1).

    Scoring is either one shared ``scheme`` or per-pair 4x4 match/mismatch
    schemes like the reference's batch_align (src/_compiled.py:504-529).
    ``lanes = p`` runs every pair whose segment ``ceil(m/p)`` fits the register
    budget in the reference layout (exact pass counts); the rest run in the
    throughput layout (identical scores and end coordinates)."""
    _require_cuda()
    L = _lib.load()
    q_off = np.asarray(q_off, dtype=np.int64)
    r_off = np.asarray(r_off, dtype=np.int64)
    n = int(q_off.shape[0] - 1)
    n_sym = scheme.n_symbols if scheme is not None else 4
    fq = _codes(flat_q, n_sym, "query")
    fr = _codes(flat_r, n_sym, "reference")
    qlen = np.diff(q_off).astype(np.int32)
    tlen = np.diff(r_off).astype(np.int32)
    res = {"score": np.zeros(n, np.int64), "ref_end": np.full(n, -1, np.int32),
           "query_end": np.full(n, -1, np.int32), "flags": np.zeros(n, np.uint8),
           "pass_stats": np.zeros((n, 2), np.int64), "lanes_used": np.zeros(n, np.int32),
           "seg_len": np.zeros(n, np.int32)}
    if n == 0:
        return res
    dev = {
        "qry": torch.from_numpy(fq if fq.size else np.zeros(1, np.uint8)).cuda(),
        "qs": torch.from_numpy(q_off[:-1].copy()).cuda(),
        "ql": torch.from_numpy(qlen).cuda(),
        "tgt": torch.from_numpy(fr if fr.size else np.zeros(1, np.uint8)).cuda(),
        "ts": torch.from_numpy(r_off[:-1].copy()).cuda(),
        "tl": torch.from_numpy(tlen).cuda(),
    }
    per_pair = scheme is None
    if per_pair:
        pp = [torch.from_numpy(np.asarray(x, dtype=np.int32)).cuda()
              for x in (match_a, mis_a, go_a, ge_a)]
        sub_t, go, ge, bias, max_sub = None, 0, 0, 0, 0
    else:
        pp = [None] * 4
        sub_t = torch.from_numpy(scheme.as_array()).cuda()
        go, ge, bias, max_sub = scheme.gap_open, scheme.gap_extend, scheme.bias, scheme.max_score
    out = {k: torch.full((n,), 0 if k == "score" else -1, dtype=torch.int32, device="cuda")
           for k in ("score", "ref_end", "query_end")}
    out["flags"] = torch.zeros(n, dtype=torch.uint8, device="cuda")
    pstats = torch.zeros((n, 2), dtype=torch.int64, device="cuda") if stats else None
    kid = _kernel_id(kernel)
    st = _stream()

    def run(width_, lanes_, order_np, n_dev=None, max_q=None, min_q=None):
        order_t = torch.from_numpy(order_np.astype(np.int32)).cuda()
        n_ = 0 if n_dev is not None else int(order_np.shape[0])
        _lib.check(L.sw_pairs_align(width_, lanes_, kid, _ptr(dev["qry"]), _ptr(dev["qs"]),
                                    _ptr(dev["ql"]), _ptr(dev["tgt"]), _ptr(dev["ts"]),
                                    _ptr(dev["tl"]), _ptr(order_t), n_, _ptr(n_dev), min_q, max_q,
                                    _ptr(sub_t), n_sym, go, ge, bias, max_sub,
                                    *[_ptr(x) for x in pp], _ptr(out["score"]),
                                    _ptr(out["ref_end"]) if coords else None,
                                    _ptr(out["query_end"]) if coords else None,
                                    _ptr(out["flags"]), None, _ptr(pstats), st))
        return order_t

    # partition: reference layout where it fits, throughput layout elsewhere
    groups = []
    if lanes:
        Lp = (qlen.astype(np.int64) + lanes - 1) // lanes
        fits = np.zeros(n, bool)
        try:
            _lib.plan_query(1, n_sym, width, lanes)
            fits = Lp <= 32
        except _lib.SwError:
            pass
        if fits.any():
            groups.append((lanes, np.flatnonzero(fits)))
        if (~fits).any():
            groups.append((0, np.flatnonzero(~fits)))
    else:
        groups.append((0, np.arange(n)))
    keep = []
    for ln, idx in groups:
        # length-sorted processing order: query length (segment), then target length
        idx = idx[np.lexsort((-tlen[idx], -qlen[idx]))]
        mq, nq = int(qlen[idx].max()), int(qlen[idx].min())
        keep.append(run(width, ln, idx, max_q=mq, min_q=nq))
        plan = _lib.plan_query(max(1, mq), n_sym, width, ln)
        res["lanes_used"][idx] = plan.lanes
        res["seg_len"][idx] = np.maximum(1, (qlen[idx] + plan.lanes - 1) // plan.lanes)
    if width == 16:
        lst = torch.empty(n, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        _lib.check(L.sw_collect_flagged(_ptr(out["flags"]), n, _lib.FLAG_RESCUE, _ptr(lst),
                                        _ptr(cnt), st))
        mq = int(qlen.max())
        _lib.check(L.sw_pairs_align(32, 0, kid, _ptr(dev["qry"]), _ptr(dev["qs"]),
                                    _ptr(dev["ql"]), _ptr(dev["tgt"]), _ptr(dev["ts"]),
                                    _ptr(dev["tl"]), _ptr(lst), 0, _ptr(cnt), 0, mq,
                                    _ptr(sub_t), n_sym, go, ge, bias, max_sub,
                                    *[_ptr(x) for x in pp], _ptr(out["score"]),
                                    _ptr(out["ref_end"]) if coords else None,
                                    _ptr(out["query_end"]) if coords else None,
                                    _ptr(out["flags"]), None, _ptr(pstats), st))
    for k, v in out.items():
        res[k] = v.cpu().numpy()
    res["score"] = res["score"].astype(np.int64)
    if stats:
        res["pass_stats"] = pstats.cpu().numpy()
    return res


def align_starts(flat_q, q_off, flat_r, r_off, scheme: ScoringScheme, score, ref_end,
                 query_end, width: int = 16) -> tuple[np.ndarray, np.ndarray]:
    """Start coordinates of optimal local alignments (the
    reference has no traceback): for each pair with its exact
    ``score`` and first-max end cell, the 0-based ``(ref_start, query_start)`` of
    the optimal alignment ending there that is shortest in the reference (ties:
    largest query start); ``(-1, -1)`` for score 0 or an unlocated end (-2).

    Device method: one pairs launch over the reversed prefixes
    ``query[query_end::-1]`` / ``ref[ref_end::-1]``, each preceded by a run of
    ``r = ceil((score + 1) / 127)`` copies of an extra symbol X scoring +127
    against itself and -127 against everything else. Every alignment through all
    r X pairs scores ``127 r + (anchored score from the end pair)`` and every other
    alignment scores below ``127 r``, so the first cell reaching
    ``127 r + score`` in the kernel's reference-major order is the alignment's
    first pair -- the same rule as the oracle's anchored reverse DP
    (oracle/sw_oracle.c swo_start_coords). Exactness is checked: the launch must
    return exactly ``127 r + score``."""
    q_off = np.asarray(q_off, dtype=np.int64)
    r_off = np.asarray(r_off, dtype=np.int64)
    sc = np.asarray(score, dtype=np.int64)
    re_ = np.asarray(ref_end, dtype=np.int64)
    qe = np.asarray(query_end, dtype=np.int64)
    n = int(q_off.shape[0] - 1)
    rs = np.full(n, -1, np.int32)
    qs = np.full(n, -1, np.int32)
    sel = np.nonzero((sc > 0) & (re_ >= 0) & (qe >= 0))[0]
    if sel.size == 0:
        return rs, qs
    A = scheme.n_symbols
    if A + 1 > 32:
        raise _lib.SwError(_lib.SW_ENOTSUP, "start coordinates need an alphabet of <= 31 symbols")
    if np.any(re_[sel] >= np.diff(r_off)[sel]) or np.any(qe[sel] >= np.diff(q_off)[sel]):
        raise ValueError("end cell outside the sequences")
    fq = _codes(flat_q, A, "query")
    fr = _codes(flat_r, A, "reference")
    reps = (sc[sel] + 1 + 126) // 127

    def reversed_ext(flat, off, end):
        lens = reps + end[sel] + 1
        o = np.zeros(sel.size + 1, np.int64)
        np.cumsum(lens, out=o[1:])
        pair = np.repeat(np.arange(sel.size), lens)
        k = np.arange(int(o[-1]), dtype=np.int64) - o[pair]
        src = off[sel][pair] + end[sel][pair] - (k - reps[pair])
        out = np.where(k < reps[pair], A, flat[np.clip(src, 0, max(flat.size - 1, 0))])
        return out.astype(np.uint8), o

    xq, xq_off = reversed_ext(fq, q_off, qe)
    xr, xr_off = reversed_ext(fr, r_off, re_)
    mat = np.full((A + 1, A + 1), -127, dtype=np.int64)
    mat[:A, :A] = scheme.as_array()
    mat[A, A] = 127
    xs = ScoringScheme.from_array(mat, scheme.gap_open, scheme.gap_extend)
    # pairs kernel for queries the warp kernels hold in 32 bits, the strip pipeline
    # (one launch per pair) beyond
    xql = np.diff(xq_off)
    got = {"score": np.zeros(sel.size, np.int64), "ref_end": np.zeros(sel.size, np.int64),
           "query_end": np.zeros(sel.size, np.int64)}
    short = np.nonzero(xql <= 1024)[0]
    if short.size:
        lq, lr = xql[short], np.diff(xr_off)[short]
        sq = np.concatenate([xq[xq_off[i]:xq_off[i + 1]] for i in short])
        sr = np.concatenate([xr[xr_off[i]:xr_off[i + 1]] for i in short])
        o = pairs_align(sq, np.concatenate([[0], np.cumsum(lq)]), sr,
                        np.concatenate([[0], np.cumsum(lr)]), scheme=xs, width=width)
        for key in got:
            got[key][short] = o[key]
    for i in np.nonzero(xql > 1024)[0]:
        o = align_long(xq[xq_off[i]:xq_off[i + 1]], xr[xr_off[i]:xr_off[i + 1]], xs, width=width)
        for key in got:
            got[key][i] = o[key]
    want = 127 * reps + sc[sel]
    if not np.array_equal(got["score"].astype(np.int64), want):
        bad = int(np.nonzero(got["score"] != want)[0][0])
        raise ValueError(f"pair {int(sel[bad])}: no alignment from the end cell reaches the score")
    rs[sel] = (re_[sel] - (got["ref_end"] - reps)).astype(np.int32)
    qs[sel] = (qe[sel] - (got["query_end"] - reps)).astype(np.int32)
    return rs, qs


def batch_align(kernel_id, p, flat_q, q_off, flat_r, r_off, match_a, mis_a, go_a, ge_a):
    """src/_compiled.py:504-529: per-pair 4x4 DNA schemes, kernel_id 0 = lazy-F with
    early exit, 1 = lazy-F full, 2 = scan. Returns ``(scores int64[n], overflow
    uint8[n], counters int64[n, 7])`` like the reference. Lazy-F runs in
    reference-mirroring mode so, for pairs whose reference layout fits
    (ceil(m/p) <= 32), the counters equal the reference's exactly."""
    kernel = {0: "lazyf-mirror", 1: "lazyf-noexit-mirror", 2: "scan"}[int(kernel_id)]
    ref_kernel = {0: "lazyf", 1: "lazyf-noexit", 2: "scan"}[int(kernel_id)]
    r = pairs_align(flat_q, q_off, flat_r, r_off, kernel=kernel, lanes=int(p), match_a=match_a,
                    mis_a=mis_a, go_a=go_a, ge_a=ge_a, stats=True, coords=False)
    n = r["score"].shape[0]
    tl = np.diff(np.asarray(r_off, dtype=np.int64))
    counters = np.zeros((n, 7), dtype=np.int64)
    for t in range(n):
        counters[t] = counters_from_stats(ref_kernel, int(tl[t]), int(r["seg_len"][t]),
                                          int(r["lanes_used"][t]), int(r["pass_stats"][t, 0]),
                                          int(r["pass_stats"][t, 1]))
    return (r["score"], (r["flags"] & _lib.FLAG_REF_OVERFLOW).astype(np.uint8), counters)


def batch_align_coords(kernel_id, p, flat_q, q_off, flat_r, r_off, match_a, mis_a, go_a, ge_a):
    """batch_align plus end coordinates: ``(scores, overflow, ref_end, query_end)``."""
    kernel = {0: "lazyf", 1: "lazyf-noexit", 2: "scan"}[int(kernel_id)]
    r = pairs_align(flat_q, q_off, flat_r, r_off, kernel=kernel, lanes=int(p), match_a=match_a,
                    mis_a=mis_a, go_a=go_a, ge_a=ge_a)
    return (r["score"], (r["flags"] & _lib.FLAG_REF_OVERFLOW).astype(np.uint8), r["ref_end"],
            r["query_end"])


def batch_oracle_scores(flat_q, q_off, flat_r, r_off, match_a, mis_a, go_a, ge_a):
    """src/_compiled.py:491-501 (exact scores; here computed by the device scan kernel)."""
    return batch_align(2, 0, flat_q, q_off, flat_r, r_off, match_a, mis_a, go_a, ge_a)[0]


def scan_lanes(f, d, width: int = 32) -> np.ndarray:
    """Device weighted max-scan over the lanes of each row of ``f`` (weighted_max_scan,
    src/kernels.py:188-201)."""
    _require_cuda()
    f = np.ascontiguousarray(np.atleast_2d(np.asarray(f, dtype=np.uint16)))
    n, p = f.shape
    fd = torch.from_numpy(f.view(np.int16)).cuda()
    dd = torch.from_numpy(np.minimum(np.asarray(d, dtype=np.int64), 2**31 - 1).astype(np.int32)).cuda()
    out = torch.empty_like(fd)
    _lib.check(_lib.load().sw_scan_lanes(width, p, _ptr(fd), _ptr(dd), n, _ptr(out), _stream()))
    return out.cpu().numpy().view(np.uint16)


class PairsBatch:
    """Device form of ``batch_align`` for large batches of one scheme (config 3):
    the reference's serial pair loop (src/_compiled.py:504-529) becomes one
    striped-kernel launch over every pair (per-pair profiles built inside the
    kernel) plus a device-counted 32-bit re-run of the rare 16-bit wrap-guard hits.

    ``upload(...)`` makes the batch device-resident (``run`` then times the
    alignment alone); ``run_host(...)`` is the end-to-end form for pinned host
    buffers: chunks are copied on a copy stream while the previous chunk is
    aligned, and the scores (and coordinates) come back per chunk. Results are
    exact either way (tests/test_gpu_fullsize.py)."""

    def __init__(self, scheme: ScoringScheme, kernel: str = "scan", coords: bool = False,
                 lanes: int = 0):
        self.scheme = as_scheme(scheme)
        self.kernel = kernel
        self.kid = _kernel_id(kernel)
        self.coords = coords
        self.lanes = lanes
        self.launches = 0
        self.sub = None

    def _meta(self, q_off, r_off):
        q_off = np.asarray(q_off, dtype=np.int64)
        r_off = np.asarray(r_off, dtype=np.int64)
        return (q_off[:-1], np.diff(q_off).astype(np.int32), r_off[:-1],
                np.diff(r_off).astype(np.int32))

    def upload(self, flat_q, q_off, flat_r, r_off) -> None:
        """Copy a CSR batch to the device (outside any timed region)."""
        _require_cuda()
        qs, ql, ts, tl = self._meta(q_off, r_off)
        n = int(ql.shape[0])
        self.n = n
        self.qlen_rng = (int(ql.min()) if n else 0, int(ql.max()) if n else 0)
        f = lambda a, dt=None: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        self.dev = {"q": f(_codes(flat_q, self.scheme.n_symbols, "query")), "qs": f(qs),
                    "ql": f(ql), "t": f(_codes(flat_r, self.scheme.n_symbols, "reference")),
                    "ts": f(ts), "tl": f(tl)}
        self.out = self._outputs(n)

    def _outputs(self, n: int) -> dict:
        o = {k: torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
             for k in ("score", "ref_end", "query_end")}
        o["flags"] = torch.zeros(max(n, 1), dtype=torch.uint8, device="cuda")
        o["_list"] = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        o["_cnt"] = torch.zeros(1, dtype=torch.int64, device="cuda")
        return o

    def _launch(self, dev: dict, out: dict, n: int, qmin: int, qmax: int) -> None:
        L = _lib.load()
        sch = self.scheme
        if self.sub is None:
            self.sub = torch.from_numpy(sch.as_array()).cuda()
        st = _stream()
        co = self.coords
        args = (_ptr(dev["q"]), _ptr(dev["qs"]), _ptr(dev["ql"]), _ptr(dev["t"]), _ptr(dev["ts"]),
                _ptr(dev["tl"]))
        tail = (_ptr(self.sub), sch.n_symbols, sch.gap_open, sch.gap_extend, sch.bias,
                sch.max_score, None, None, None, None, _ptr(out["score"]),
                _ptr(out["ref_end"]) if co else None, _ptr(out["query_end"]) if co else None,
                _ptr(out["flags"]), None, None, st)
        _lib.check(L.sw_pairs_align(16, self.lanes, self.kid, *args, None, n, None, qmin, qmax,
                                    *tail))
        # 16-bit wrap-guard hits: collected and re-run in 32 bits on the device
        _lib.check(L.sw_collect_flagged(_ptr(out["flags"]), n, _lib.FLAG_RESCUE,
                                        _ptr(out["_list"]), _ptr(out["_cnt"]), st))
        _lib.check(L.sw_pairs_align(32, 0, self.kid, *args, _ptr(out["_list"]), 0,
                                    _ptr(out["_cnt"]), 0, qmax, *tail))
        self.launches += 3

    def run(self) -> dict:
        """Align the uploaded batch; device results (score, ref_end, query_end, flags)."""
        self._launch(self.dev, self.out, self.n, *self.qlen_rng)
        return self.out

    @staticmethod
    def pin_host(flat_q, q_off, flat_r, r_off, packed2bit: bool = False) -> dict:
        """Pinned host copies of a CSR batch (the e2e input form). ``packed2bit``: the
        residues as four 2-bit codes per byte (``formats.pack_2bit``; DNA codes 0..3,
        fixed-length batches), a quarter of the bytes over the host link; the device
        expands each chunk (``sw_unpack_2bit``)."""
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        if packed2bit:
            from .formats import pack_2bit

            return {"q2": pin(pack_2bit(flat_q)), "q_off": np.asarray(q_off, np.int64),
                    "t2": pin(pack_2bit(flat_r)), "r_off": np.asarray(r_off, np.int64)}
        return {"q": pin(np.asarray(flat_q, np.uint8)), "q_off": np.asarray(q_off, np.int64),
                "t": pin(np.asarray(flat_r, np.uint8)), "r_off": np.asarray(r_off, np.int64)}

    def prepare_host(self, host: dict, n_chunks: int = 16) -> None:
        """Per-chunk metadata (chunk-relative starts, lengths) in pinned memory and
        double-buffered device chunk buffers; done once per batch, outside timing."""
        q_off, r_off = host["q_off"], host["r_off"]
        n = int(q_off.shape[0] - 1)
        n_chunks = max(1, min(n_chunks, n))
        qlen, tlen = np.diff(q_off), np.diff(r_off)
        # fixed-length batches (reads against equal windows, config 3): starts and lengths
        # follow from the two lengths, so they are generated on the device once instead of
        # being copied per chunk (the H2D carries residues only)
        self.uniform = n > 0 and bool((qlen == qlen[0]).all() and (tlen == tlen[0]).all())
        self.packed2 = "q2" in host
        bounds = [n * c // n_chunks for c in range(n_chunks + 1)]
        if self.packed2:
            if not self.uniform:
                raise ValueError("2-bit packed input needs a fixed-length batch")
            # chunks start on a packed byte (and a 4-byte code word) of both streams
            bounds = sorted({min(n, b // 32 * 32) for b in bounds[:-1]} | {n})
        chunks = []
        for a, b in zip(bounds[:-1], bounds[1:]):
            qs = q_off[a:b] - q_off[a]
            ts = r_off[a:b] - r_off[a]
            meta = None if self.uniform else torch.from_numpy(np.concatenate([
                qs.view(np.int32), ts.view(np.int32), np.diff(q_off[a:b + 1]).astype(np.int32),
                np.diff(r_off[a:b + 1]).astype(np.int32)])).pin_memory()
            ql = np.diff(q_off[a:b + 1])
            chunks.append((a, b, int(q_off[a]), int(q_off[b]), int(r_off[a]), int(r_off[b]), meta,
                           int(ql.min()) if b > a else 0, int(ql.max()) if b > a else 0))
        self.chunks = chunks
        mq = max(c[3] - c[2] for c in chunks)
        mt = max(c[5] - c[4] for c in chunks)
        mn = max(c[1] - c[0] for c in chunks)
        self.bufs = [{"q": torch.empty(max(mq, 1) + 16, dtype=torch.uint8, device="cuda"),
                      "t": torch.empty(max(mt, 1) + 16, dtype=torch.uint8, device="cuda"),
                      "q2": torch.empty((max(mq, 1) + 3) // 4 if self.packed2 else 1,
                                        dtype=torch.uint8, device="cuda"),
                      "t2": torch.empty((max(mt, 1) + 3) // 4 if self.packed2 else 1,
                                        dtype=torch.uint8, device="cuda"),
                      "meta": torch.empty(6 * mn, dtype=torch.int32, device="cuda"),
                      "out": self._outputs(mn)} for _ in range(2)]
        self.host_out = {k: torch.empty(n, dtype=torch.int32).pin_memory()
                         for k in (("score", "ref_end", "query_end") if self.coords else ("score",))}
        self.host_out["flags"] = torch.empty(n, dtype=torch.uint8).pin_memory()
        if self.uniform:
            idx = torch.arange(mn, dtype=torch.int64, device="cuda")
            self.umeta = {"qs": idx * int(qlen[0]), "ts": idx * int(tlen[0]),
                          "ql": torch.full((mn,), int(qlen[0]), dtype=torch.int32, device="cuda"),
                          "tl": torch.full((mn,), int(tlen[0]), dtype=torch.int32, device="cuda")}
        self.copy_stream = torch.cuda.Stream()
        self.h2d_bytes = int((host["q2"].numel() + host["t2"].numel()) if self.packed2 else
                             (host["q"].numel() + host["t"].numel()
                              + sum(c[6].numel() * 4 for c in chunks if c[6] is not None)))
        self.d2h_bytes = int(sum(v.numel() * v.element_size() for v in self.host_out.values()))

    def run_host(self, host: dict) -> dict:
        """End to end from pinned host buffers: chunk c+1 is copied while chunk c is
        aligned; per-chunk results are copied back into pinned host arrays. Returns
        the host result tensors (valid after a synchronize)."""
        cur = torch.cuda.current_stream()
        cp = self.copy_stream
        ready = [torch.cuda.Event() for _ in self.chunks]
        freed = [torch.cuda.Event() for _ in range(2)]
        for c, (a, b, qa, qb, ta, tb, meta, qmin, qmax) in enumerate(self.chunks):
            buf = self.bufs[c & 1]
            n = b - a
            with torch.cuda.stream(cp):
                if c >= 2:
                    cp.wait_event(freed[c & 1])  # the chunk that used this buffer is done
                if self.packed2:  # qa, ta are multiples of 4 (chunk bounds of 32 pairs)
                    nq2, nt2 = (qb - qa + 3) // 4, (tb - ta + 3) // 4
                    buf["q2"][:nq2].copy_(host["q2"][qa // 4:qa // 4 + nq2], non_blocking=True)
                    buf["t2"][:nt2].copy_(host["t2"][ta // 4:ta // 4 + nt2], non_blocking=True)
                else:
                    buf["q"][: qb - qa].copy_(host["q"][qa:qb], non_blocking=True)
                    buf["t"][: tb - ta].copy_(host["t"][ta:tb], non_blocking=True)
                if meta is not None:
                    buf["meta"][: 6 * n].copy_(meta, non_blocking=True)
                if self.packed2:  # expanded on the copy stream, beside the previous chunk's alignment
                    L = _lib.load()
                    _lib.check(L.sw_unpack_2bit(_ptr(buf["q2"]), qb - qa, _ptr(buf["q"]), cp.cuda_stream))
                    _lib.check(L.sw_unpack_2bit(_ptr(buf["t2"]), tb - ta, _ptr(buf["t"]), cp.cuda_stream))
                    self.launches += 2
                ready[c].record(cp)
            cur.wait_event(ready[c])
            if meta is None:
                u = self.umeta
                dev = {"q": buf["q"], "t": buf["t"], "qs": u["qs"][:n], "ts": u["ts"][:n],
                       "ql": u["ql"][:n], "tl": u["tl"][:n]}
            else:
                m = buf["meta"]
                dev = {"q": buf["q"], "t": buf["t"], "qs": m[0:2 * n], "ts": m[2 * n:4 * n],
                       "ql": m[4 * n:5 * n], "tl": m[5 * n:6 * n]}
            o = buf["out"]
            self._launch(dev, o, n, qmin, qmax)
            for k, v in self.host_out.items():
                v[a:b].copy_(o[k][:n], non_blocking=True)
            freed[c & 1].record(cur)
        return self.host_out
