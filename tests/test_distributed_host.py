"""Host-side logic of the row-partitioned solver (CPU): partition, local CSR
blocks, halo mirror ranges, and the torch.distributed communicator over gloo
with two processes."""

import os

import numpy as np
import pytest

import paper_2105_07544_b200 as mk
from paper_2105_07544_b200 import distributed as dd

from conftest import random_csr


@pytest.mark.parametrize("n,P", [(1024, 2), (1024, 3), (64000, 8), (8_000_000, 8), (2_250_000, 7), (130, 2)])
def test_row_partition(n, P):
    s = dd.row_partition(n, P)
    assert s[0] == 0 and s[-1] == n and len(s) == P + 1
    assert all(s[p] % 64 == 0 for p in range(P))
    assert all(s[p + 1] > s[p] for p in range(P))
    # within one alignment block of the ideal floor(p n / P) split
    assert all(abs(s[p] - p * n // P) < 64 for p in range(P))


def test_row_partition_rejects_tiny():
    with pytest.raises(mk.DimensionMismatchError):
        dd.row_partition(100, 3)


def _blocks(A, P):
    s = dd.row_partition(A.n, P)
    return s, [dd.local_csr(A, s[p], s[p + 1]) for p in range(P)]


@pytest.mark.parametrize("preset,nx,P", [("Laplace3D", 12, 3), ("BentPipe2D", 40, 4), ("Stretched2D", 24, 2)])
def test_local_csr_reassembles_bit_exact(preset, nx, P):
    A = mk.generate_stencil(mk.ProblemSpec(preset, nx))
    s, blocks = _blocks(A, P)
    rp = [np.zeros(1, np.int64)]
    base = 0
    cols, vals = [], []
    for p, (lrp, lci, lv) in enumerate(blocks):
        rp.append(lrp[1:] + base)
        base += lrp[-1]
        cols.append(lci + s[p])
        vals.append(lv)
    assert np.array_equal(np.concatenate(rp), A.row_ptr)
    assert np.array_equal(np.concatenate(cols), A.col_idx)
    assert np.concatenate(vals).tobytes() == A.values.tobytes()


def _check_mirrors_cover(A, P):
    s = dd.row_partition(A.n, P)
    reach = dd.operator_reach(A, s)
    mirrors = [dd.mirror_ranges(s, reach, p) for p in range(P)]
    owner = np.searchsorted(np.array(s[1:]), np.arange(A.n), side="right")
    for q in range(P):
        a, b = A.row_ptr[s[q]], A.row_ptr[s[q + 1]]
        need = np.unique(A.col_idx[a:b])
        need = need[(need < s[q]) | (need >= s[q + 1])]
        for c in need:
            p = owner[c]
            lo, hi = mirrors[p][0][q], mirrors[p][1][q]
            assert lo <= c - s[p] < hi, (q, c, p, lo, hi)
        # ranges are 64-aligned at the low end and stay inside the block
        for p in range(P):
            lo, hi = mirrors[p][0][q], mirrors[p][1][q]
            assert lo % 64 == 0 and 0 <= lo <= hi <= s[p + 1] - s[p]
            if p == q:
                assert lo == hi == 0


@pytest.mark.parametrize("preset,nx,P", [("Laplace3D", 16, 3), ("Laplace3D", 16, 8), ("BentPipe2D", 64, 5),
                                         ("Stretched2D", 40, 4), ("UniFlow2D", 32, 2)])
def test_mirror_ranges_cover_every_halo_column(preset, nx, P):
    A = mk.generate_stencil(mk.ProblemSpec(preset, nx))
    _check_mirrors_cover(A, P)
    # the stencil reach is the matrix-free operator's; the CSR one agrees or is smaller
    A.use_stencil = False
    s = dd.row_partition(A.n, P)
    st = dd.operator_reach(A, s)
    A2 = mk.CsrMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    cs = dd.operator_reach(A2, s)
    assert all(c[0] <= t[0] and c[1] <= t[1] for c, t in zip(cs, st))


def test_mirror_ranges_random_far_columns(rng):
    A, _ = random_csr(mk, rng, 300, density=0.05)
    _check_mirrors_cover(A, 3)


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = dd.TorchComm()
        got = c.exchange({"rank": rank, "h": bytes([rank]) * 64})
        assert [g["rank"] for g in got] == list(range(world))
        sums = c.allreduce_host([np.float32(0.1) * (rank + 1), 2.0 ** -30 * rank, rank])
        n = 200
        s = dd.row_partition(n, world, align=8)
        local = torch.arange(s[rank], s[rank + 1], dtype=torch.float64)
        glob = torch.zeros(n, dtype=torch.float64)
        c.allgather_rows(local, glob, s)
        q.put((rank, [float(v) for v in sums], bool(torch.equal(glob, torch.arange(n, dtype=torch.float64)))))
    finally:
        dist.destroy_process_group()


def test_torch_comm_over_gloo_two_ranks():
    import socket

    import torch.multiprocessing as tmp

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    # identical, rank-ordered sums on both ranks
    assert out[0][1] == out[1][1]
    assert out[0][1][0] == float(np.float32(0.1) * 1 + np.float32(0.1) * 2)
    assert all(o[2] for o in out)
