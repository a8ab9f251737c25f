"""Host logic of the sharded path (-m "not gpu"): world size 2 over gloo on CPU.
Segment maps and fold come from the oracle here; on GPUs they are the library's
kernels (tests/test_gpu_parity.py::test_segment_maps_fold)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W
from paper_1210_5093_b200 import multi_gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, n, cuts, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = W.get(name)
        a = w.automaton
        x = w.input(n)
        bounds = np.array([0] + list(cuts) + [n], np.uint64)
        od = oracle.Dfa(a.table, a.q0, a.accepting)
        imax = max(1, od.imax())
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        seg = x[lo:hi]

        def segment_map(lookahead):
            row = np.full(imax, 0xFFFF, np.uint16)
            if lookahead < 0:
                row[0] = od.run(seg)
            else:
                assert lookahead == x[lo - 1]
                row[:], _ = od.chunk_map(x, lo, hi, imax)
            return torch.from_numpy(row.view(np.int16).copy())

        def fold(rows, lookahead):
            r = rows.numpy().view(np.uint16)
            return od.fold(x, bounds, imax, int(r[0][0]), r[1:])

        m = multi_gpu.SegmentMatcher(rank, world, dist, torch.from_numpy(seg[-1:].copy()), segment_map, fold)
        got = [m.step() for _ in range(2)]
        q.put((rank, got, od.run(x), m.lookahead))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,n,cuts", [("random", 200_000, [123_457]), ("keyword", 150_000, [1]),
                                         ("tiny", 4096, [4000]), ("protein", 100_000, [50_000])])
def test_two_ranks_gloo(name, n, cuts):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, n, cuts, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, expect, la in res:
        assert got == [expect, expect], (rank, got, expect)
        x = W.get(name).input(n)
        assert la == [-1, int(x[cuts[0] - 1])]
