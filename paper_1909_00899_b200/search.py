"""Database search: one query against a length-binned, sharded target database.

The reference has no database driver; its batch entry point is a serial loop
over pairs (batch_align, src/_compiled.py:504-529) and the runner aligns one
pair at a time (src/runner.py:113-159). This module is the B200 replacement for
that caller side of the hot path:

* ``PackedDb``: the host-side database format -- uint8 residue codes, int64
  starts, int32 lengths, a length-descending processing order (so the G
  alignments that share a warp have near-equal length) and global target ids,
  in pinned memory so uploads run at PCIe/C2C speed;
* ``shard``: balanced partition of the targets over ranks (round-robin over the
  length-sorted order, so every rank gets the same cell count to within one
  target);
* ``DatabaseSearch``: device buffers + the launch sequence per query (profile
  build, 16-bit striped kernel, device-side 32-bit rescue, top-k);
* ``merge_topk``: the cross-rank top-k merge (one all_gather of k records per
  rank over NCCL -- the only collective of the path).

Top-k order: score descending, then global target id ascending.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .align import DeviceProfile, _ptr, _stream, build_profile_arrays, rescue_long
from .scoring import ScoringScheme

RECORD_FIELDS = ("score", "target_id", "ref_end", "query_end")


@dataclass
class PackedDb:
    codes: torch.Tensor  # uint8 [total residues] (pinned host or device)
    start: torch.Tensor  # int64 [n]
    length: torch.Tensor  # int32 [n]
    order: torch.Tensor  # int32 [n] length-descending processing order
    ids: torch.Tensor  # int64 [n] global target ids

    @property
    def n(self) -> int:
        return int(self.length.shape[0])

    @property
    def residues(self) -> int:
        return int(self.length.sum())

    def nbytes(self) -> int:
        return sum(int(t.numel() * t.element_size())
                   for t in (self.codes, self.start, self.length, self.order, self.ids))


def shard(offsets: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Global target ids owned by `rank`: round-robin over the length-descending order."""
    lens = np.diff(np.asarray(offsets, dtype=np.int64))
    by_len = np.argsort(-lens, kind="stable")
    return np.sort(by_len[rank::world])


def shard_pairs(n_pairs: int, rank: int, world: int) -> tuple[int, int]:
    """Pair batch sharding (config 3): rank r owns the contiguous range
    [a, b) of the pairs; pairs are independent, so no exchange is needed."""
    a = n_pairs * rank // world
    b = n_pairs * (rank + 1) // world
    return a, b


def gather_pairs(local: torch.Tensor, n_pairs: int, group=None) -> torch.Tensor:
    """Per-pair results of contiguous pair shards (shard_pairs) gathered on every
    rank in global pair order: one all_gather of each rank's [b - a, ...] block,
    padded to the largest shard (NCCL on device tensors, gloo on host tensors).
    The only exchange config 3 has, and an optional one."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return local[:n_pairs]
    world = dist.get_world_size(group)
    dev = local.device
    if dist.get_backend(group) == "gloo":
        local = local.cpu()
    sizes = [b - a for a, b in (shard_pairs(n_pairs, r, world) for r in range(world))]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:n] for p, n in zip(parts, sizes)]).to(dev)


PACKED_FILES = ("codes", "start", "length", "order", "ids")


def save_packed(path: str, packed: PackedDb, alphabet: str | None = None) -> None:
    """Write a PackedDb as a directory of .npy arrays (memory-mappable) plus meta.json."""
    import json
    import os

    os.makedirs(path, exist_ok=True)
    for name in PACKED_FILES:
        np.save(os.path.join(path, name + ".npy"), getattr(packed, name).numpy())
    meta = {"format": "b200-swscan-packed-db", "version": 1, "n": packed.n,
            "residues": packed.residues, "alphabet": alphabet}
    with open(os.path.join(path, "meta.json"), "w") as fh:
        json.dump(meta, fh)


def load_packed(path: str, pin: bool = True) -> tuple[PackedDb, dict]:
    """Read a directory written by save_packed (arrays land in pinned host memory)."""
    import json
    import os

    with open(os.path.join(path, "meta.json")) as fh:
        meta = json.load(fh)
    if meta.get("format") != "b200-swscan-packed-db":
        raise ValueError(f"{path}: not a packed database")

    def t(name):  # one copy from the memory-mapped file into (pinned) host memory
        a = np.load(os.path.join(path, name + ".npy"), mmap_mode="r")
        x = torch.empty(a.shape, dtype=torch.from_numpy(np.empty(0, a.dtype)).dtype,
                        pin_memory=pin and torch.cuda.is_available())
        x.numpy()[...] = a
        return x

    packed = PackedDb(*(t(name) for name in PACKED_FILES))
    if packed.n != meta["n"]:
        raise ValueError(f"{path}: {packed.n} targets, meta says {meta['n']}")
    return packed, meta


def pack(db: np.ndarray, offsets: np.ndarray, ids: np.ndarray | None = None,
         pin: bool = True) -> PackedDb:
    """Pack the targets `ids` (default: all) of a CSR database into a PackedDb,
    physically in length-descending order (ties by global id): every contiguous
    range of targets is then a load-balanced launch on its own, and the
    processing order is the identity."""
    offsets = np.asarray(offsets, dtype=np.int64)
    if ids is None:
        ids = np.arange(offsets.shape[0] - 1, dtype=np.int64)
    ids = np.asarray(ids, dtype=np.int64)
    lens0 = offsets[ids + 1] - offsets[ids]
    ids = ids[np.argsort(-lens0, kind="stable")]
    lens = (offsets[ids + 1] - offsets[ids]).astype(np.int64)
    start = np.zeros(ids.shape[0], dtype=np.int64)
    if ids.shape[0]:
        np.cumsum(lens[:-1], out=start[1:])
    codes = np.empty(int(lens.sum()), dtype=np.uint8)
    step = 1 << 16  # gather in blocks of targets to bound the index array
    for a in range(0, ids.shape[0], step):
        b = min(ids.shape[0], a + step)
        ln = lens[a:b]
        idx = np.repeat(offsets[ids[a:b]] - start[a:b], ln) + np.arange(
            int(start[a]), int(start[a]) + int(ln.sum()), dtype=np.int64)
        codes[int(start[a]): int(start[a]) + int(ln.sum())] = db[idx]
    order = np.arange(ids.shape[0], dtype=np.int32)

    def t(a):
        x = torch.from_numpy(np.ascontiguousarray(a))
        return x.pin_memory() if pin and torch.cuda.is_available() else x

    return PackedDb(t(codes if codes.size else np.zeros(1, np.uint8)), t(start),
                    t(lens.astype(np.int32)), t(order), t(ids))


class DatabaseSearch:
    """Device-resident database + per-query launch sequence.

    ``upload(packed)`` copies a PackedDb into device buffers (async on the
    current stream); ``align(query)`` runs profile build + 16-bit striped kernel
    + device-side 32-bit rescue; ``topk(k)`` returns the k best records of this
    rank as a device int64 tensor [k, 4] (score, target_id, ref_end, query_end).

    ``coords``: ``"all"`` locates the end coordinates of every target;
    ``"topk"`` locates them for every target that can enter the top ``k``: the
    launch processes a strided sample of the database first (every 16th target
    outside the longest 1/8, so the sample finishes quickly), and the warp that
    completes the sample raises a coordinate floor to the k-th best of its
    exact scores (``floor_sample`` of ``sw_db_align``); every later task reads
    the floor. Every target scoring >= the floor (a superset of the final top
    k) gets exact coordinates, the others report (-2, -2). Scores are exact in
    both modes. One launch, no host sync.
    """

    SAMPLE_STRIDE = int(os.environ.get("SWB_SAMPLE_STRIDE", "16"))  # coordinate-floor sample: every n-th target

    def __init__(self, scheme: ScoringScheme, kernel: str = "scan", lanes: int = 0,
                 coords: str = "all", k: int = 100):
        if coords not in ("all", "topk"):
            raise ValueError(f"coords must be 'all' or 'topk', got {coords!r}")
        self.scheme = scheme
        self.kernel = kernel
        self.lanes = lanes
        self.coords = coords
        self.k = k
        self.kid = _lib.KERNEL_IDS[kernel]
        self.dev: PackedDb | None = None
        self.out: dict | None = None
        self.prof: DeviceProfile | None = None
        self.launches = 0
        # streamed input: a chunk later than this aborts the feed and the jobs it
        # held are re-run after the copies (0 = the library default, 2 s)
        self.feed_timeout_ns = int(float(os.environ.get("SWB_FEED_TIMEOUT_MS", "0")) * 1e6)

    def _ensure_buffers(self, packed: PackedDb) -> None:
        n = packed.n
        if self.dev is None or self.dev.n != n or self.dev.codes.numel() < packed.codes.numel():
            self.dev = PackedDb(*(torch.empty_like(x, device="cuda") for x in
                                  (packed.codes, packed.start, packed.length, packed.order,
                                   packed.ids)))
            self.out = {
                "score": torch.empty(n, dtype=torch.int32, device="cuda"),
                "ref_end": torch.empty(n, dtype=torch.int32, device="cuda"),
                "query_end": torch.empty(n, dtype=torch.int32, device="cuda"),
                "flags": torch.empty(n, dtype=torch.uint8, device="cuda"),
                "_rescue": (torch.empty(max(n, 1), dtype=torch.int32, device="cuda"),
                            torch.zeros(1, dtype=torch.int64, device="cuda")),
                "_refeed": (torch.empty(max(n, 1), dtype=torch.int32, device="cuda"),
                            torch.zeros(1, dtype=torch.int64, device="cuda")),
                "_floor": torch.zeros(1, dtype=torch.int32, device="cuda"),
            }

    def upload(self, packed: PackedDb) -> None:
        self._ensure_buffers(packed)
        for dst, src in zip((self.dev.codes, self.dev.start, self.dev.length, self.dev.order,
                             self.dev.ids),
                            (packed.codes, packed.start, packed.length, packed.order, packed.ids)):
            dst[: src.numel()].copy_(src, non_blocking=True)

    def set_query(self, query) -> DeviceProfile:
        self.prof = build_profile_arrays(query, self.scheme, self.lanes)
        self.prof.ensure32()
        self.plan16, self.prof16 = self.prof.for_kernel(self.kernel)
        self.launches += 2
        return self.prof

    def rebuild_profile(self) -> None:
        """Re-run the profile kernels for the current query (device-resident)."""
        L = _lib.load()
        p = self.prof
        _lib.check(L.sw_profile_build(C.byref(self.plan16), _ptr(p.query), _ptr(p.sub), p.bias,
                                      _ptr(self.prof16), _stream()))
        self.launches += 1

    def _launch16(self, n: int, floor: bool, sample: int = 0,
                  order: torch.Tensor | None = None, feed: tuple | None = None) -> None:
        """16-bit striped kernel over the n database slots; ``order``: processing
        order of the job ids; ``floor``: gate coordinates on the floor buffer;
        ``sample`` > 0: the launch raises the floor from the first ``sample`` jobs
        of its processing order; ``feed`` = (d_arrived, jobs per chunk, epoch):
        streamed input (see sw_db_opts_t)."""
        L = _lib.load()
        p, d, o, sch = self.prof, self.dev, self.out, self.scheme
        opts = None
        if floor or feed:
            opts = _lib.DbOpts(d_coord_floor=o["_floor"].data_ptr() if floor else None,
                               floor_sample=sample, floor_k=self.k)
            if feed:
                opts.d_arrived, opts.arrive_jobs, opts.arrive_epoch = (feed[0].data_ptr(),
                                                                       feed[1], feed[2])
                opts.arrive_timeout_ns = self.feed_timeout_ns
        _lib.check(L.sw_db_align(C.byref(self.plan16), _ptr(self.prof16), self.kid, sch.gap_open,
                                 sch.gap_extend, p.bias, p.max_sub, _ptr(d.codes), _ptr(d.start),
                                 _ptr(d.length), _ptr(order), n, None, _ptr(o["score"]),
                                 _ptr(o["ref_end"]), _ptr(o["query_end"]), _ptr(o["flags"]),
                                 None, None, C.byref(opts) if opts else None, _stream()))
        self.launches += 1

    def _sampled_order(self, n: int, region: int | None = None) -> tuple[torch.Tensor | None, int]:
        """Processing order for a launch over n length-sorted jobs in coords='topk'
        mode: (sample, then the rest in length order), and the sample size. The
        sample is every SAMPLE_STRIDE-th job of [region/8, region) (region = n by
        default; the first chunk when the input is streamed). (None, 0) when every
        target gets coordinates."""
        if self.coords != "topk" or self.plan16.width != 16 or self.kernel != "scan":
            return None, 0
        region = n if region is None else min(region, n)
        cache = getattr(self, "_orders", {})
        if (n, region) not in cache:
            idx = torch.arange(n, dtype=torch.int32, device="cuda")
            pick = torch.zeros(n, dtype=torch.bool, device="cuda")
            pick[region // 8:region:self.SAMPLE_STRIDE] = True
            cnt = int(pick.sum().item())
            if cnt < self.k:
                cache[(n, region)] = (None, 0)
            else:
                cache[(n, region)] = (torch.cat([idx[pick], idx[~pick]]).contiguous(), cnt)
            self._orders = cache
        return cache[(n, region)]

    def _rescue(self, n: int) -> None:
        L = _lib.load()
        p, d, o, sch = self.prof, self.dev, self.out, self.scheme
        if p.long32:  # query beyond the 32-bit warp kernels: strip-pipeline rescues
            rescue_long(p, d.codes, d.start, d.length, o, n)
            return
        st = _stream()
        lst, cnt = o["_rescue"]
        _lib.check(L.sw_collect_flagged(_ptr(o["flags"]), n, _lib.FLAG_RESCUE, _ptr(lst),
                                        _ptr(cnt), st))
        _lib.check(L.sw_db_align(C.byref(p.plan32), _ptr(p.prof32), self.kid, sch.gap_open,
                                 sch.gap_extend, p.bias, p.max_sub, _ptr(d.codes), _ptr(d.start),
                                 _ptr(d.length), _ptr(lst), 0, _ptr(cnt), _ptr(o["score"]),
                                 _ptr(o["ref_end"]), _ptr(o["query_end"]), _ptr(o["flags"]),
                                 None, None, None, st))
        self.launches += 2

    def _refeed(self, n: int, floor: bool) -> None:
        """Re-run the jobs a streamed launch gave up on (FLAG_FEED_TIMEOUT: their
        chunk had not arrived in time) with an ordinary 16-bit launch over the
        device-collected list, after the copies are done. Without a timeout the
        list is empty and the launch exits at once (no host sync either way)."""
        L = _lib.load()
        p, d, o, sch = self.prof, self.dev, self.out, self.scheme
        st = _stream()
        lst, cnt = o["_refeed"]
        _lib.check(L.sw_collect_flagged(_ptr(o["flags"]), n, _lib.FLAG_FEED_TIMEOUT, _ptr(lst),
                                        _ptr(cnt), st))
        opts = _lib.DbOpts(d_coord_floor=o["_floor"].data_ptr()) if floor else None
        _lib.check(L.sw_db_align(C.byref(self.plan16), _ptr(self.prof16), self.kid, sch.gap_open,
                                 sch.gap_extend, p.bias, p.max_sub, _ptr(d.codes), _ptr(d.start),
                                 _ptr(d.length), _ptr(lst), 0, _ptr(cnt), _ptr(o["score"]),
                                 _ptr(o["ref_end"]), _ptr(o["query_end"]), _ptr(o["flags"]),
                                 None, None, C.byref(opts) if opts else None, st))
        self.launches += 2

    def align(self) -> dict:
        assert self.dev is not None and self.prof is not None, "upload() and set_query() first"
        n = self.dev.n
        order, sample = self._sampled_order(n)
        if sample:
            self.out["_floor"].zero_()
        self._launch16(n, floor=bool(sample), sample=sample, order=order)
        self._rescue(n)
        return self.out

    def search_streamed(self, packed: PackedDb, n_chunks: int = 64,
                        floor_from: torch.Tensor | None = None,
                        _starve_copy: bool = False) -> dict:
        """End-to-end form for a host-resident (pinned) database, one kernel launch:
        the copy stream uploads chunk c (residues, starts, lengths, ids) and then
        its arrival flag; the striped kernel, launched at once, makes each task
        wait for the chunk holding its targets, so the H2D transfer overlaps the
        alignment with no per-chunk launch tails. Requires set_query(); returns
        the result dict.

        CUDA does not promise that the copies run while the kernel does (profilers,
        CUDA_LAUNCH_BLOCKING and sanitizers serialise them): a task whose chunk is
        late by ``feed_timeout_ns`` aborts the feed, the launch flags every job it
        did not align with FLAG_FEED_TIMEOUT, and those jobs are re-run here once
        the copies are done -- results are exact either way, never silently 0."""
        assert self.prof is not None, "set_query() first"
        self._ensure_buffers(packed)
        d, o = self.dev, self.out
        n = packed.n
        if n == 0:
            return o
        cur = torch.cuda.current_stream()
        copy = self._copy_stream = getattr(self, "_copy_stream", None) or torch.cuda.Stream()
        n_chunks = max(1, min(n_chunks, n))
        cj = -(-n // n_chunks)
        cj = -(-cj // 32) * 32  # chunk boundaries on 32-job (128-byte) lines
        n_chunks = -(-n // cj)
        if getattr(self, "_arrived", None) is None or self._arrived.numel() < n_chunks:
            self._arrived = torch.zeros(max(n_chunks, 64), dtype=torch.int32, device="cuda")
            self._epoch = 0
        self._epoch += 1
        # residue ranges of the chunks (recomputed every call: O(n_chunks))
        st, ln = packed.start.numpy(), packed.length.numpy()
        chunks = [(c * cj, min(n, (c + 1) * cj), int(st[c * cj]),
                   int(st[min(n, (c + 1) * cj) - 1] + ln[min(n, (c + 1) * cj) - 1]))
                  for c in range(n_chunks)]
        marks = torch.full((n_chunks,), self._epoch, dtype=torch.int32).pin_memory()
        copy.wait_stream(cur)  # buffers may still be read by a previous step
        # launch first (its tasks wait for their chunk), then feed the chunks
        order, sample = self._sampled_order(n, region=cj)
        if sample:
            o["_floor"].zero_()
        if sample and floor_from is not None:  # a known lower bound: no sampling needed
            o["_floor"].copy_(floor_from.reshape(1))
            order, sample = None, 0
            floor_on = True
        else:
            floor_on = bool(sample)
        self._launch16(n, floor=floor_on, sample=sample, order=order,
                       feed=(self._arrived, cj, self._epoch))
        if _starve_copy:  # test hook: the copies may only start after the kernel
            copy.wait_stream(cur)
        with torch.cuda.stream(copy):
            for c, (a, b, ra, rb) in enumerate(chunks):
                d.codes[ra:rb].copy_(packed.codes[ra:rb], non_blocking=True)
                d.start[a:b].copy_(packed.start[a:b], non_blocking=True)
                d.length[a:b].copy_(packed.length[a:b], non_blocking=True)
                self._arrived[c:c + 1].copy_(marks[c:c + 1], non_blocking=True)
            d.ids[:n].copy_(packed.ids, non_blocking=True)  # for top-k only
        cur.wait_stream(copy)  # ids before topk; the copy stream's work before the next step
        self._refeed(n, floor_on)  # jobs whose chunk timed out, now that it is resident
        self._rescue(n)
        return o

    def search_large(self, packed: PackedDb, max_residues: int, n_chunks: int = 64) -> torch.Tensor:
        """Top-k over a database larger than the device buffers: passes of at most
        ``max_residues`` residues (contiguous, so each pass stays length-sorted),
        each streamed through one launch; the running top-k is merged on the
        device, and from the second pass on its k-th score is the coordinate floor
        (a lower bound of the final k-th best, so no sampling is needed).
        Returns int64 [k, 4] records (score, target_id, ref_end, query_end)."""
        assert self.prof is not None, "set_query() first"
        lens = packed.length.numpy().astype(np.int64)
        cum = np.concatenate([[0], np.cumsum(lens)])
        best, kth = None, None
        a = 0
        while a < packed.n:
            b = int(np.searchsorted(cum, cum[a] + max_residues, side="right")) - 1
            b = max(b, a + 1)  # a single target larger than the budget still runs alone
            ra, rb = int(cum[a]), int(cum[b])
            start = packed.start[a:b] - ra
            view = PackedDb(packed.codes[ra:rb], start.pin_memory() if packed.codes.is_pinned()
                            else start, packed.length[a:b], packed.order[a:b] - a,
                            packed.ids[a:b])
            self.search_streamed(view, n_chunks, floor_from=kth)
            top = self.topk(self.k)
            best = top if best is None else select_topk(torch.cat([best, top]), self.k)
            if best.shape[0] >= self.k:
                kth = best[self.k - 1, 0].to(torch.int32)
            a = b
        return best

    def topk(self, k: int = 100) -> torch.Tensor:
        """k best (score desc, global id asc) as int64 [k, 4] on the device."""
        o, d = self.out, self.dev
        self.launches += 3  # sw_topk: histogram + threshold, compaction, one-CTA sort
        return topk_records(o["score"], d.ids, o["ref_end"], o["query_end"], k)


_TOPK_WORK: dict = {}


def topk_records(score: torch.Tensor, ids: torch.Tensor, ref_end: torch.Tensor,
                 query_end: torch.Tensor, k: int) -> torch.Tensor:
    """The k best records (score desc, global id asc) as int64 [k, 4]
    (score, target_id, ref_end, query_end).  Device tensors go through the library's
    own top-k (``sw_topk``: score histogram -> threshold -> compaction -> one-CTA
    sort); host tensors (the gloo tests) through torch."""
    k = min(k, int(score.shape[0]))
    if (score.is_cuda and 1 <= k <= 1024 and score.dtype == torch.int32
            and ids.dtype == torch.int64 and ref_end.dtype == torch.int32
            and query_end.dtype == torch.int32):
        L = _lib.load()
        dev = score.device.index if score.device.index is not None else torch.cuda.current_device()
        st = torch.cuda.current_stream()
        wkey = (dev, st.cuda_stream)  # launches on one stream run in order: one scratch each
        work = _TOPK_WORK.get(wkey)
        if work is None:
            work = torch.empty(int(L.sw_topk_workspace()), dtype=torch.uint8, device=score.device)
            _TOPK_WORK[wkey] = work
        rec = torch.empty((k, 4), dtype=torch.int64, device=score.device)
        n = int(score.shape[0])
        _lib.check(L.sw_topk(score.contiguous().data_ptr(), ids.contiguous().data_ptr(),
                             ref_end.contiguous().data_ptr(), query_end.contiguous().data_ptr(),
                             n, k, rec.data_ptr(), work.data_ptr(), st.cuda_stream))
        return rec
    key = (score.to(torch.int64) << 32) | (0xFFFFFFFF - ids.to(torch.int64))
    _, idx = torch.topk(key, k, sorted=True)
    return torch.stack([score[idx].to(torch.int64), ids[idx].to(torch.int64),
                        ref_end[idx].to(torch.int64), query_end[idx].to(torch.int64)], dim=1)


def select_topk(records: torch.Tensor, k: int) -> torch.Tensor:
    """The k best of int64 [r, 4] records (score desc, target id asc)."""
    key = (records[:, 0] << 32) | (0xFFFFFFFF - (records[:, 1] & 0xFFFFFFFF))
    _, idx = torch.topk(key, min(k, records.shape[0]), sorted=True)
    return records[idx]


def merge_topk(records: torch.Tensor, k: int, group=None) -> torch.Tensor:
    """Cross-rank top-k: all_gather k records per rank (NCCL), re-select on every rank."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return records
    world = dist.get_world_size(group)
    dev = records.device
    if dist.get_backend(group) == "gloo":  # gloo collectives run on host tensors
        records = records.cpu()
    kk = torch.full((k, 4), -1, dtype=torch.int64, device=records.device)
    kk[: records.shape[0]] = records
    kk[records.shape[0]:, 0] = -1  # padding (scores are >= 0) loses every comparison
    gathered = [torch.empty_like(kk) for _ in range(world)]
    dist.all_gather(gathered, kk, group=group)
    allr = torch.cat(gathered)
    key = (allr[:, 0] << 32) | (0xFFFFFFFF - (allr[:, 1] & 0xFFFFFFFF))
    _, idx = torch.topk(key, min(k, allr.shape[0]), sorted=True)
    return allr[idx].to(dev)


def hit_starts(query, records, db: np.ndarray, offsets: np.ndarray, scheme: ScoringScheme,
               width: int = 16) -> np.ndarray:
    """Top-k hits with start coordinates: int64 [k, 6] (score, target_id, ref_end,
    query_end, ref_start, query_start). ``records`` are topk/merge_topk records;
    ``db``/``offsets`` the database CSR in global target ids. One device launch for
    all hits (align.align_starts); hits without located ends keep (-1, -1)."""
    from .align import align_starts

    rec = records.cpu().numpy() if isinstance(records, torch.Tensor) else np.asarray(records)
    rec = rec.astype(np.int64).reshape(-1, 4)
    rec = rec[rec[:, 0] >= 0]
    k = rec.shape[0]
    q = np.asarray(query, dtype=np.uint8)
    offsets = np.asarray(offsets, dtype=np.int64)
    q_off = np.arange(k + 1, dtype=np.int64) * q.size
    ids = rec[:, 1]
    lens = offsets[ids + 1] - offsets[ids]
    r_off = np.zeros(k + 1, np.int64)
    np.cumsum(lens, out=r_off[1:])
    flat_r = (np.concatenate([db[offsets[i]:offsets[i + 1]] for i in ids]) if k
              else np.zeros(0, np.uint8))
    rs, qs = align_starts(np.tile(q, k), q_off, flat_r, r_off, scheme, rec[:, 0], rec[:, 2],
                          rec[:, 3], width=width)
    return np.concatenate([rec, rs[:, None].astype(np.int64), qs[:, None].astype(np.int64)], axis=1)
