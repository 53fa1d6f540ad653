"""Multi-rank host logic on CPU (torch.distributed gloo, world size 2).

The device path of a rank needs a GPU (tests/test_gpu_slabs.py runs the same
slab code path on one GPU with device-copy halos); here: the row partition, the
per-rank input slices (local_part) and the NCCL unique-id handshake every rank
performs before gpcg_create_*_dist.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_cs_0101018_b200 import problems as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problems():
    from tests.test_gpu_parity import ragged_stencil
    return [ragged_stencil(13, 11, 3), ragged_stencil(9, 8, 4, full=False), P.c4_family(m=6),
            P.journal_bearing(12, 10)]


def _worker(rank, world, port, outq):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_cs_0101018_b200 import gpcg
    try:
        # NCCL unique id: made on rank 0, broadcast, identical everywhere
        obj = [gpcg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        res = {"id_ok": len(obj[0]) == 128 and all(i == ids[0] for i in ids), "parts": []}
        for prob in _problems():
            rows = gpcg.problem_rows(prob)
            rb, re = gpcg.partition_rows(rows, world, rank)
            loc = gpcg.local_part(prob, rb, re)
            res["parts"].append((rb, re, loc))
        outq.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def gathered():
    from paper_cs_0101018_b200 import _build
    _build.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return world, out


def test_nccl_id_handshake(gathered):
    world, out = gathered
    assert all(out[r]["id_ok"] for r in range(world))


def test_partition_covers_rows_in_rank_order(gathered):
    world, out = gathered
    probs = _problems()
    for k, prob in enumerate(probs):
        from paper_cs_0101018_b200 import gpcg
        spans = [out[r]["parts"][k][:2] for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == gpcg.problem_rows(prob)
        for a, b in zip(spans, spans[1:]):
            assert a[1] == b[0]
        sizes = [e - b for b, e in spans]
        assert max(sizes) - min(sizes) <= 1


def test_local_parts_reassemble_the_problem(gathered):
    world, out = gathered
    for k, prob in enumerate(_problems()):
        parts = [out[r]["parts"][k] for r in range(world)]
        for key in ("b", "l", "u", "x0"):
            assert np.array_equal(np.concatenate([p[2][key] for p in parts]), np.asarray(getattr(prob, key)))
        if prob.kind == "stencil2d":
            nx = prob.nx
            if prob.wx_ld:
                full = np.asarray(prob.wx)
                for rb, re, loc in parts:
                    for j in range(rb, re):
                        assert np.array_equal(loc["wx"][(j - rb) * prob.wx_ld:(j - rb) * prob.wx_ld + nx + 1],
                                              full[j * prob.wx_ld:j * prob.wx_ld + nx + 1])
            if prob.wy_ld:
                full = np.asarray(prob.wy)
                for rb, re, loc in parts:        # face rows rb..re inclusive: the shared one on both ranks
                    for f in range(rb, re + 1):
                        assert np.array_equal(loc["wy"][(f - rb) * prob.wy_ld:(f - rb) * prob.wy_ld + nx],
                                              full[f * prob.wy_ld:f * prob.wy_ld + nx])
            if prob.shift is not None:
                assert np.array_equal(np.concatenate([p[2]["shift"] for p in parts]), prob.shift)
        else:
            rp = np.asarray(prob.row_ptr)
            for rb, re, loc in parts:
                assert loc["row_ptr"][0] == 0 and len(loc["row_ptr"]) == re - rb + 1
                assert np.array_equal(loc["row_ptr"], rp[rb:re + 1] - rp[rb])
                assert np.array_equal(loc["col"], np.asarray(prob.col)[rp[rb]:rp[re]])
                # the band a rank's columns reach stays within ranks r-1, r, r+1 (gpcg.h requirement)
                assert loc["col"].min() >= 0 and loc["col"].max() < prob.n


def test_partition_rows_edge_cases():
    from paper_cs_0101018_b200 import _build, gpcg
    _build.build()
    assert gpcg.partition_rows(10, 3, 0) == (0, 4)
    assert gpcg.partition_rows(10, 3, 1) == (4, 7)
    assert gpcg.partition_rows(10, 3, 2) == (7, 10)
    assert gpcg.partition_rows(8000, 8, 7) == (7000, 8000)
    assert gpcg.partition_rows(5, 0, 0) == (0, 0)          # invalid -> empty
    for total in (1, 7, 64, 1001):
        for parts in (1, 2, 3, 8):
            spans = [gpcg.partition_rows(total, parts, k) for k in range(parts)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
