"""Multi-rank host logic on CPU (gloo, world size 2): database sharding and the
top-k merge that bench.py runs over NCCL. Scores come from the CPU oracle."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1909_00899_b200 import search, workloads as W


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, out_q)
    except BaseException as exc:  # surface failures instead of hanging the parent
        out_q.put((rank, "error", repr(exc), None))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, world, out_q):
    if True:
        from oracle import oracle as O

        w = W.config2(n_targets=400)
        ids = search.shard(w.offsets, rank, world)
        packed = search.pack(w.db, w.offsets, ids, pin=False)
        # the shard's own packed layout must reproduce each target exactly
        assert sorted(packed.ids.tolist()) == sorted(ids.tolist())
        lens = packed.length.numpy()
        assert (lens[:-1] >= lens[1:]).all(), "packed physically in length-descending order"
        for j in (0, len(ids) // 2, len(ids) - 1):
            g = int(packed.ids[j])
            a = packed.codes[int(packed.start[j]): int(packed.start[j]) + int(packed.length[j])]
            assert (a.numpy() == w.db[w.offsets[g]: w.offsets[g + 1]]).all()
        off = np.concatenate([[0], np.cumsum(packed.length.numpy())]).astype(np.int64)
        sc, re_, qe = O.db_scalar(w.query, packed.codes.numpy(), off, w.scheme.as_array(), 11, 1)
        local = search.topk_records(torch.from_numpy(sc), packed.ids, torch.from_numpy(re_),
                                    torch.from_numpy(qe), 25)
        merged = search.merge_topk(local, 25)
        # config 3: each rank generates only its own pair range and aligns it; the
        # optional result gather restores global pair order on every rank
        n3 = 3000
        a, b = search.shard_pairs(n3, rank, world)
        w3 = W.config3(n_pairs=n3, start=a, stop=b)
        s3, r3, q3 = O.batch_scalar(w3.flat_q, w3.q_off, w3.flat_r, w3.r_off,
                                    sub=w3.scheme.as_array(), go=6, ge=1)
        local3 = torch.from_numpy(np.stack([s3, r3, q3], axis=1).astype(np.int32))
        gathered = search.gather_pairs(local3, n3)
        out_q.put((rank, ids, int(packed.residues), merged.numpy(), gathered.numpy()))


def test_shard_and_topk_merge_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for r in res:
        assert not (isinstance(r[1], str) and r[1] == "error"), r[2]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    w = W.config2(n_targets=400)
    all_ids = np.sort(np.concatenate([r[1] for r in res]))
    assert (all_ids == np.arange(w.n_targets)).all(), "shards must partition the database"
    residues = [r[2] for r in res]
    assert abs(residues[0] - residues[1]) <= int(np.diff(w.offsets).max())
    # every rank holds the same merged top-k, equal to the single-process top-k
    from oracle import oracle as O

    sc, re_, qe = O.db_scalar(w.query, w.db, w.offsets, w.scheme.as_array(), 11, 1)
    want = search.topk_records(torch.from_numpy(sc), torch.arange(w.n_targets),
                               torch.from_numpy(re_), torch.from_numpy(qe), 25).numpy()
    for r in res:
        assert (r[3] == want).all()
    w3 = W.config3(n_pairs=3000)
    s3, r3, q3 = O.batch_scalar(w3.flat_q, w3.q_off, w3.flat_r, w3.r_off,
                                sub=w3.scheme.as_array(), go=6, ge=1)
    want3 = np.stack([s3, r3, q3], axis=1).astype(np.int32)
    for r in res:
        assert (r[4] == want3).all(), "gathered config-3 shards == single-process batch"
    # order: score desc, then id asc among ties
    assert all((a[0] > b[0]) or (a[0] == b[0] and a[1] < b[1]) for a, b in zip(want, want[1:]))
