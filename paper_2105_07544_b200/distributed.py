"""Row-partitioned multi-GPU solves: one rank per GPU.

The reference is single-process; the B200 build adds one parallel strategy,
a contiguous row-block partition of the system across the GPUs of a box:

* rank p owns global rows [starts[p], starts[p+1]) (``row_partition``: the
  deterministic floor(p*n/P) split rounded down to 64-row boundaries, so
  every rank's rows start on a 256/512-byte line);
* its operator is the row block: a stencil with a row offset (applied
  matrix-free) or the local CSR rows with column indices shifted to the
  rank's origin (``local_csr``);
* inside a restart cycle ONE persistent kernel per rank does everything:
  its CTAs write their CGS2 partial sums straight into every rank's partial
  buffer and the boundary rows of w'' straight into the neighbours' global
  x buffers (P2P stores through CUDA-IPC-mapped pointers over NVLink), meet
  the other ranks at a system-scope counter barrier, and reduce all ranks'
  partials in one fixed order, so every rank holds bit-identical Arnoldi
  coefficients and runs the same Givens update (no NCCL call inside the
  cycle, no host round trip);
* once per restart / refinement two small device kernels do the rest over
  the same peer memory and arrival counters: ``mpk_comm_push_rows`` stores
  the rank's x rows into its global-length buffer and the mirror rows into
  the neighbours' (the explicit residual reads its halo there), and
  ``mpk_comm_reduce_ctl`` sums r.r, r_low.r_low, b.b and the "x moved" flag
  over the ranks in rank order; the host then reads one control block, as
  on one GPU (no pickling, no NCCL, no full-x allgather).

Two communicators implement ``Comm``: :class:`TorchComm` (one process per
GPU under torchrun, NCCL/gloo for the per-restart collectives and for the
IPC-handle exchange) and :class:`ThreadComm` (P virtual ranks sharing ONE
GPU, one Python thread each, concurrent kernels on separate streams) used by
the tests, since this build's GPU runs have a single device.
"""

from __future__ import annotations

import ctypes
import dataclasses
import threading

import numpy as np

from . import _lib
from . import device as D
from .engine import OFF_BN2, OFF_CHANGED, OFF_RN2, OFF_RN2_LOW, CycleWorkspace, Readout, sqrt_in

OFF_TIMEOUT = OFF_RN2 + 20   # int32 set by mpk_comm_reduce_ctl when a cross-rank barrier timed out
from .errors import PrecisionMismatchError, DimensionMismatchError, ZeroRightHandSideError
from .gmres import ConvergenceReport, CycleState, HistoryEntry, SolverConfig, detect_loss_of_accuracy
from .multiprecision import IrConfig
from .precision import Precision
from .sparse import CsrMatrix

__all__ = ["row_partition", "operator_reach", "mirror_ranges", "local_csr", "LocalSystem", "ThreadComm",
           "TorchComm", "dist_gmres_restarted", "dist_gmres_ir", "run_virtual_ranks"]

ALIGN = 64
MAX_RANKS = 8


# ---------------------------------------------------------------------------
# host-side partition logic (pure numpy; tested on CPU)
# ---------------------------------------------------------------------------

def row_partition(n: int, nranks: int, align: int = ALIGN) -> list:
    """starts[0..P]: rank p owns rows [starts[p], starts[p+1]).  floor(p*n/P)
    rounded down to a multiple of `align`; every rank non-empty."""
    if nranks < 1 or nranks > MAX_RANKS:
        raise ValueError("1 <= nranks <= %d" % MAX_RANKS)
    starts = [min(n, (p * n // nranks) // align * align) for p in range(nranks)] + [n]
    if any(starts[p + 1] <= starts[p] for p in range(nranks)):
        raise DimensionMismatchError("%d rows cannot be split into %d non-empty %d-row-aligned blocks"
                                     % (n, nranks, align))
    return starts


def _stencil_reach(stencil) -> int:
    nx = stencil.nx
    return {"Laplace3D": nx * nx, "Stretched2D": nx + 1}.get(stencil.preset, nx)


def operator_reach(A: CsrMatrix, starts: list) -> list:
    """Per rank q: (below, above) = how far q's rows reach outside their own
    block (max row - col, max col - row, clipped at 0)."""
    P = len(starts) - 1
    if A.stencil is not None:
        h = _stencil_reach(A.stencil)
        return [(h, h)] * P
    rows = np.repeat(np.arange(A.n, dtype=np.int64), np.diff(A.row_ptr))
    off = A.col_idx - rows
    out = []
    for q in range(P):
        a, b = A.row_ptr[starts[q]], A.row_ptr[starts[q + 1]]
        seg = off[a:b]
        below = int(max(0, -seg.min())) if seg.size else 0
        above = int(max(0, seg.max())) if seg.size else 0
        out.append((below, above))
    return out


def mirror_ranges(starts: list, reach: list, rank: int, align: int = ALIGN):
    """Local row ranges [lo[q], hi[q]) of `rank`'s block that rank q reads in
    its SpMV (q != rank), rounded outward to `align` and clipped to the
    block; empty ranges are (0, 0)."""
    P = len(starts) - 1
    r0, r1 = starts[rank], starts[rank + 1]
    lo = [0] * MAX_RANKS
    hi = [0] * MAX_RANKS
    for q in range(P):
        if q == rank:
            continue
        below, above = reach[q]
        a = max(r0, starts[q] - below)
        b = min(r1, starts[q + 1] + above)
        if a >= b:
            continue
        la = (a - r0) // align * align
        lb = min(r1 - r0, -(-(b - r0) // align) * align)
        lo[q], hi[q] = la, lb
    return lo, hi


def local_csr(A: CsrMatrix, r0: int, r1: int):
    """(row_ptr, col_idx, values) of rows [r0, r1) with columns relative to
    r0 (int64 host arrays; the device copy is int32)."""
    a, b = int(A.row_ptr[r0]), int(A.row_ptr[r1])
    rp = A.row_ptr[r0:r1 + 1] - a
    ci = A.col_idx[a:b] - r0
    return rp, ci, A.values[a:b]


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------

class _ThreadShared:
    def __init__(self, nranks):
        self.nranks = nranks
        self.barrier = threading.Barrier(nranks)
        self.slots = [None] * nranks


class ThreadComm:
    """P virtual ranks on one GPU, one Python thread each (tests)."""

    def __init__(self, shared: _ThreadShared, rank: int):
        self.sh, self.rank, self.size = shared, rank, shared.nranks
        self.ctas = max(1, int(D.lib().mpk_sm_count()) // self.size)   # all ranks co-resident
        self.ipc = False

    def exchange(self, obj) -> list:
        self.sh.slots[self.rank] = obj
        self.sh.barrier.wait()
        out = list(self.sh.slots)
        self.sh.barrier.wait()
        return out

    def allreduce_host(self, vals: list) -> list:
        allv = self.exchange(list(vals))
        return [_ordered_sum([v[i] for v in allv]) for i in range(len(vals))]

    def allgather_rows(self, local, glob, starts):
        """glob[starts[q]:starts[q+1]] = rank q's `local` for every q."""
        D.sync()
        tensors = self.exchange(local)
        for q, t in enumerate(tensors):
            glob[starts[q]:starts[q + 1]].copy_(t[: starts[q + 1] - starts[q]])
        D.sync()
        self.sh.barrier.wait()   # nobody overwrites `local` before every peer copied it


class TorchComm:
    """One process per GPU (torchrun); torch.distributed for the per-restart
    collectives, CUDA IPC for the in-kernel peer pointers."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.rank, self.size = dist.get_rank(), dist.get_world_size()
        self.ctas = 0
        self.ipc = True
        if D.torch().cuda.is_available():   # host-only (gloo) tests have no device to map
            self.check_peers()

    def check_peers(self):
        """Every rank must be able to map every other rank's memory (P2P over
        NVLink); refuse loudly otherwise instead of faulting in the kernel."""
        t = D.torch()
        dev = t.cuda.current_device()
        devs = self.exchange(dev)
        lib = D.lib()
        for q, pd in enumerate(devs):
            ok = int(lib.mpk_can_access_peer(dev, pd))
            if ok != 1:
                raise RuntimeError("rank %d (cuda:%d) cannot access rank %d's device cuda:%d peer-to-peer"
                                   % (self.rank, dev, q, pd))

    def exchange(self, obj) -> list:
        from .engine import HOST_STATS

        HOST_STATS["host_collectives"] += 1
        out = [None] * self.size
        self.dist.all_gather_object(out, obj)
        return out

    def allreduce_host(self, vals: list) -> list:
        allv = self.exchange(list(vals))   # numpy scalars keep their precision
        return [_ordered_sum([v[i] for v in allv]) for i in range(len(vals))]

    def allgather_rows(self, local, glob, starts):
        t = D.torch()
        P = self.size
        c = max(starts[q + 1] - starts[q] for q in range(P))
        send = t.zeros(c, dtype=local.dtype, device=local.device)
        send[: local.shape[0]].copy_(local)
        recv = [t.empty(c, dtype=local.dtype, device=local.device) for _ in range(P)]
        self.dist.all_gather(recv, send)
        for q in range(P):
            glob[starts[q]:starts[q + 1]].copy_(recv[q][: starts[q + 1] - starts[q]])


def _ordered_sum(vals):
    """Rank-order sum in the values' own type (identical on every rank)."""
    acc = vals[0]
    for v in vals[1:]:
        acc = acc + v
    return acc


# ---------------------------------------------------------------------------
# per-rank device state
# ---------------------------------------------------------------------------

class _PeerBuffers:
    """Partial buffer, arrival counter, epoch and global-length x buffer of
    one cycle precision, with every rank's pointers."""

    def __init__(self, comm, prec: Precision, n_global: int):
        lib = D.lib()
        self.comm = comm
        sv = prec.dtype.itemsize
        self.nxg = D.ld_for(n_global) + ALIGN
        sizes = {"part": int(lib.mpk_comm_part_bytes(prec.code)), "xbar": 64, "epoch": 64,
                 "xg": self.nxg * sv}
        self.own = {}
        for k, nb in sizes.items():
            p = ctypes.c_void_p()
            _lib.check(lib.mpk_dev_alloc(nb, ctypes.byref(p)))
            self.own[k] = p.value
        if comm.ipc:
            mine = {}
            for k in ("part", "xbar", "xg"):
                h = ctypes.create_string_buffer(64)
                _lib.check(lib.mpk_ipc_get(ctypes.c_void_p(self.own[k]), h))
                mine[k] = h.raw
            allh = comm.exchange(mine)
            self.peers = {k: [] for k in ("part", "xbar", "xg")}
            self._opened = []
            for q, hs in enumerate(allh):
                for k in ("part", "xbar", "xg"):
                    if q == comm.rank:
                        self.peers[k].append(self.own[k])
                        continue
                    p = ctypes.c_void_p()
                    _lib.check(lib.mpk_ipc_open(ctypes.create_string_buffer(hs[k], 64), ctypes.byref(p)))
                    self.peers[k].append(p.value)
                    self._opened.append(p.value)
        else:
            allp = comm.exchange({k: self.own[k] for k in ("part", "xbar", "xg")})
            self.peers = {k: [allp[q][k] for q in range(comm.size)] for k in ("part", "xbar", "xg")}
            self._opened = []
        # keep the peers' buffers alive until everyone is done with ours
        comm.exchange(None)

    def close(self):
        lib = D.lib()
        for p in self._opened:
            lib.mpk_ipc_close(ctypes.c_void_p(p))
        self.comm.exchange(None)
        for p in self.own.values():
            lib.mpk_dev_free(ctypes.c_void_p(p))
        self.own = {}


class LocalSystem:
    """Rank-local view of a global system: row block, local operator (fp64
    and fp32), mirror ranges and the peer buffers of both cycle precisions."""

    def __init__(self, comm, A: CsrMatrix, A_low: CsrMatrix | None = None):
        self.comm = comm
        self.A_global = A
        self.n_global = A.n
        self.starts = row_partition(A.n, comm.size)
        self.r0, self.r1 = self.starts[comm.rank], self.starts[comm.rank + 1]
        self.n = self.r1 - self.r0
        self.reach = operator_reach(A, self.starts)
        self.mir_lo, self.mir_hi = mirror_ranges(self.starts, self.reach, comm.rank)
        self.ops = {}
        for prec, M in ((A.precision, A), (None if A_low is None else A_low.precision, A_low)):
            if M is not None:
                self.ops[prec] = self._local_op(M)
        self._peers = {}
        self._ws = {}

    def _local_op(self, M: CsrMatrix):
        d = _lib.MpkMatrix()
        d.dtype = M.precision.code
        d.n = self.n
        d.row0 = self.r0
        keep = []
        if M.stencil is not None and M.use_stencil:
            s = M.stencil
            d.kind = _lib.STENCIL
            d.nnz = 0
            d.preset = _lib.PRESET_IDS[s.preset]
            d.nx = s.nx
            d.diffusion, d.velocity = s.diffusion, s.velocity
            d.convection, d.stretch = s.convection, s.stretch
        else:
            rp, ci, vals = local_csr(M, self.r0, self.r1)
            trp = D.to_device(rp.astype(np.int32))
            tci = D.to_device(ci.astype(np.int32))
            tv = D.to_device(np.ascontiguousarray(vals))
            keep = [trp, tci, tv]
            d.kind = _lib.CSR
            d.nnz = int(vals.shape[0])
            d.row_ptr, d.col_idx, d.values = D.ptr(trp), D.ptr(tci), D.ptr(tv)
        return d, keep

    def op(self, prec: Precision):
        if prec not in self.ops:
            raise DimensionMismatchError("no %s operator for this rank" % prec.value)
        return self.ops[prec][0]

    def peers(self, prec: Precision) -> _PeerBuffers:
        if prec not in self._peers:
            self._peers[prec] = _PeerBuffers(self.comm, prec, self.n_global)
        return self._peers[prec]

    def workspace(self, m: int, prec: Precision) -> CycleWorkspace:
        key = (m, prec)
        if key not in self._ws:
            self._ws[key] = CycleWorkspace(self.n, m, prec)   # private (not the per-device cache)
        return self._ws[key]

    def comm_struct(self, prec: Precision) -> _lib.MpkComm:
        pb = self.peers(prec)
        c = _lib.MpkComm()
        c.rank, c.nranks, c.ctas = self.comm.rank, self.comm.size, self.comm.ctas
        c.row0 = self.r0
        for q in range(self.comm.size):
            c.part[q] = pb.peers["part"][q]
            c.xbar[q] = pb.peers["xbar"][q]
            c.xg[q] = pb.peers["xg"][q]
            c.mir_lo[q], c.mir_hi[q] = self.mir_lo[q], self.mir_hi[q]
        c.epoch = pb.own["epoch"]
        return c

    def prepare(self, precs, m: int, M=None, cycle_prec: Precision | None = None):
        """Create every device resource a solve needs BEFORE its first
        cross-rank kernel: peer buffers of each precision set (cudaMalloc +
        CUDA-IPC open), the cycle workspace, the preconditioner descriptor.
        Allocation / IPC mapping can wait for the device to go idle, and a
        peer's persistent kernel spinning at the cross-rank barrier never
        does, so a rank that allocates lazily while its peers spin
        deadlocks until the barrier's 20 s timeout.  The first call per
        resource set ends with one host barrier (every rank is ready); later
        solves on the same system do no host collective."""
        key = (tuple(sorted(p.value for p in precs)), m, id(M) if M is not None else None, cycle_prec)
        done = getattr(self, "_prepared", set())
        if key in done:
            return
        for p in precs:
            self.peers(p)
        if cycle_prec is not None:
            self.workspace(m, cycle_prec)
            self.comm_struct(cycle_prec)
            if M is not None:
                self.diag_precond(M, cycle_prec)
        D.sync()
        self.comm.exchange(None)
        done.add(key)
        self._prepared = done

    def diag_precond(self, M, prec: Precision) -> _lib.MpkPrecond:
        """mpk_precond of a block-Jacobi(1) right preconditioner (a diagonal
        scaling, applied inside the row-partitioned cycle kernel): `lu` points
        at row0 of the GLOBAL diagonal, so the halo rows the SpMV reads
        (local indices below 0 or past n) find their a_ii as well."""
        key = ("diag", id(M), prec)
        got = getattr(self, "_diag_cache", {}).get(key)
        if got is not None:
            return got[0]
        if getattr(M, "kind", None) != "jacobi" or M.data.block_size != 1:
            raise ValueError("row-partitioned cycles support block Jacobi with 1x1 blocks (or no preconditioner)")
        if M.precision is not prec or M.n != self.n_global:
            raise PrecisionMismatchError("preconditioner must be built on the global matrix in the cycle precision")
        nat = M.native()
        d = _lib.MpkPrecond()
        d.kind = _lib.PC_JACOBI
        d.dtype = prec.code
        d.n = self.n
        d.block = 1
        d.lu = nat.lu + self.r0 * prec.dtype.itemsize
        d.piv = nat.piv + self.r0 * 4
        if not hasattr(self, "_diag_cache"):
            self._diag_cache = {}
        self._diag_cache[key] = (d, M)
        return d

    def close(self):
        for pb in self._peers.values():
            pb.close()
        self._peers = {}


# ---------------------------------------------------------------------------
# distributed cycle workspace: CycleWorkspace's interface, global semantics
# ---------------------------------------------------------------------------

class _DistWs:
    def __init__(self, sysm: LocalSystem, m: int, prec: Precision):
        self.s = sysm
        self.ws = sysm.workspace(m, prec)
        self.prec = prec
        self._comm_struct = sysm.comm_struct(prec)
        self._push_prec = prec

    def residual(self, prec, b, x, r, r_low=None):
        """r = b - A x on the rank's rows.  x (precision `prec`) goes into the
        rank's global-length buffer of that precision set and its mirror rows
        into the neighbours' (mpk_comm_push_rows, P2P + cross-rank barrier);
        the residual kernel reads its halo there."""
        s = self.s
        lib = D.lib()
        cs = s.comm_struct(prec)
        _lib.check(lib.mpk_comm_push_rows(ctypes.addressof(cs), prec.code, s.n, D.ptr(x), D.stream()))
        xv = s.peers(prec).own["xg"] + s.r0 * prec.dtype.itemsize
        d = s.op(prec)
        _lib.check(lib.mpk_residual(ctypes.byref(d), D.ptr(b), xv, D.ptr(r),
                                    self.ws.at(OFF_RN2), D.ptr(r_low) if r_low is not None else None,
                                    self.ws.at(OFF_RN2_LOW) if r_low is not None else None,
                                    self.ws.ws.ptr, D.stream()))
        self._push_prec = prec

    def bnorm2(self, b, prec):
        self.ws.bnorm2(b, prec)

    def cycle(self, prec, r0, rnorm2_off, x0, x_out, steps_cap, exit_tol, norm_scale, rule, orth="cgs2",
              M=None):
        ws = self.ws
        d = ws.desc
        mat = self.s.op(prec)
        ws._pins = [mat, self._comm_struct]
        d.A = ctypes.pointer(mat)
        d.M = None
        if M is not None:
            md = self.s.diag_precond(M, prec)
            ws._pins.append(md)
            d.M = ctypes.pointer(md)
        d.dtype = prec.code
        d.m = ws.m
        d.steps_cap = int(steps_cap)
        d.rule = _lib.RULE_U if rule == "u" else _lib.RULE_NU
        d.exit_tol = float(exit_tol)
        d.norm_scale = float(norm_scale) if norm_scale is not None else -1.0
        d.n = ws.n
        d.ld = ws.ld
        d.V = D.ptr(ws.V)
        d.r0 = D.ptr(r0)
        d.rnorm2 = ws.at(rnorm2_off)
        d.x0 = D.ptr(x0)
        d.x_out = D.ptr(x_out)
        d.work = D.ptr(ws.work)
        d.hess = D.ptr(ws.hess)
        d.ws = ws.ws.ptr
        d.ctl = ws.ctl_ptr
        d.nranks = self.s.comm.size
        d.flags = ws.flags | (16 if orth == "dcgs2" else 0)
        d.comm = ctypes.pointer(self._comm_struct)
        _lib.check(D.lib().mpk_cycle_run(ctypes.byref(d), D.stream()))

    def read(self, rn2_dtype=np.float64, with_cycle=True, bn2_dtype=None) -> Readout:
        """Sum r.r, r_low.r_low, b.b and the 'moved' flag over the ranks on
        the device (mpk_comm_reduce_ctl, rank order, in place in the slots the
        next cycle reads), then the one control-block read of a restart."""
        prec = self._push_prec
        rt = np.dtype(rn2_dtype)
        bt = np.dtype(bn2_dtype or rn2_dtype)
        code = lambda dt: _lib.F64 if dt == np.float64 else _lib.F32  # noqa: E731
        cs = self.s.comm_struct(prec)
        _lib.check(D.lib().mpk_comm_reduce_ctl(ctypes.addressof(cs), prec.code, self.ws.at(OFF_RN2),
                                               code(rt), code(bt), D.stream()))
        out = self.ws.read(rn2_dtype=rn2_dtype, with_cycle=with_cycle)
        raw = self.ws.host.numpy()
        if int(np.frombuffer(raw, dtype=np.int32, count=1, offset=OFF_TIMEOUT)[0]) or \
                (with_cycle and int(np.frombuffer(raw, dtype=np.int32, count=6, offset=0)[5])):
            raise RuntimeError("row-partitioned solve: a rank missed the cross-GPU barrier (timeout)")
        self._bn2 = float(np.frombuffer(raw, dtype=bt, count=1, offset=OFF_BN2)[0])
        return out

    def bn2(self) -> float:
        return self._bn2


# ---------------------------------------------------------------------------
# drivers (same bookkeeping as gmres.gmres_restarted / multiprecision.gmres_ir)
# ---------------------------------------------------------------------------

def _local_vec(sysm: LocalSystem, v, dtype):
    """Rank-local slice of a global vector (numpy or tensor) as a device tensor."""
    if D.shape(v) == (sysm.n_global,):
        v = v[sysm.r0:sysm.r1]
    elif D.shape(v) != (sysm.n,):
        raise DimensionMismatchError("vector is neither global (%d) nor local (%d) length"
                                     % (sysm.n_global, sysm.n))
    return D.to_device(v, dtype).clone()


def dist_gmres_restarted(sysm: LocalSystem, b, x0, cfg: SolverConfig, norm_baseline=None,
                         explicit_restart_on_loss=True, phase=None, M=None):
    """gmres_restarted (reference gmres.py:221-308) on the rank's rows; the
    report (identical on every rank) carries the rank-local x.  M: None or a
    block-Jacobi(1) preconditioner built on the global matrix (right
    preconditioning, applied inside the cycle kernel)."""
    prec = cfg.precision
    if cfg.m + 1 > 52:
        raise ValueError("row-partitioned cycles support m <= 51")
    if cfg.basis_precision != "working":
        raise ValueError("row-partitioned cycles keep the basis in the working precision")
    t = D.torch()
    bd = _local_vec(sysm, b, prec.torch_dtype)
    x = _local_vec(sysm, x0, prec.torch_dtype)
    r = D.empty(sysm.n, prec.torch_dtype)
    sysm.prepare([prec], cfg.m, M, prec)   # after every allocation of this solve
    ws = _DistWs(sysm, cfg.m, prec)
    if phase is None:
        phase = "double" if prec is Precision.binary64 else "single"
    ws.bnorm2(bd, prec)
    ws.residual(prec, bd, x, r)
    first = ws.read(rn2_dtype=prec.dtype, with_cycle=False)
    if sqrt_in(prec, ws.bn2()) == 0.0:
        raise ZeroRightHandSideError("right-hand side is identically zero")
    own = sqrt_in(prec, first.rn2)
    scale = own if norm_baseline is None else float(norm_baseline)
    history = [HistoryEntry(0, phase, None, own / scale if scale else 0.0)]
    if own == 0.0:
        return ConvergenceReport(True, 0, 0, 0.0, history, False, x, scale, phase_iters={phase: 0})
    total = restarts = 0
    loss = converged = False
    explicit = own / scale
    while True:
        if explicit <= cfg.rtol:
            converged = True
            break
        remaining = cfg.max_iters - total
        if remaining <= 0 or restarts >= cfg.max_restarts:
            break
        cap = max(1, min(cfg.m, remaining))
        ws.cycle(prec, r, OFF_RN2, x, x, cap, cfg.rtol, scale, cfg.breakdown_rule, cfg.orthogonalization, M)
        ws.residual(prec, bd, x, r)
        out = ws.read(rn2_dtype=prec.dtype)
        state = CycleState(out.steps, out.implicit, scale, out.breakdown)
        for i, rel in enumerate(out.implicit):
            history.append(HistoryEntry(total + i + 1, phase, rel, None))
        total += out.steps
        restarts += 1
        explicit = sqrt_in(prec, out.rn2) / scale
        if out.steps:
            history[-1] = dataclasses.replace(history[-1], explicit_relres=explicit)
        now = detect_loss_of_accuracy(state, explicit, cfg.rtol)
        loss = loss or now
        if now and not explicit_restart_on_loss:
            break
    return ConvergenceReport(converged, total, restarts, explicit, history, loss, x, scale,
                             phase_iters={phase: total})


def dist_gmres_ir(sysm: LocalSystem, b, x0, cfg: IrConfig, M=None):
    """gmres_ir (reference multiprecision.py:120-233) on the rank's rows.
    M: None or a block-Jacobi(1) preconditioner (fp32, global matrix)."""
    prec, low = cfg.outer_precision, cfg.inner.precision
    if prec is not Precision.binary64 or low is not Precision.binary32:
        raise ValueError("the device refinement runs fp32 inside fp64")
    if cfg.inner.m + 1 > 52:
        raise ValueError("row-partitioned cycles support m <= 51")
    if cfg.inner.basis_precision != "working":
        raise ValueError("row-partitioned cycles keep the basis in the working precision")
    t = D.torch()
    n = sysm.n
    bd = _local_vec(sysm, b, t.float64)
    x = _local_vec(sysm, x0, t.float64)
    r = D.empty(n, t.float64)
    r32 = D.empty(n, t.float32)
    u32 = D.empty(n, t.float32)
    zeros32 = D.zeros(n, t.float32)
    sysm.prepare([prec, low], cfg.inner.m, M, low)   # after every allocation of this solve
    ws = _DistWs(sysm, cfg.inner.m, low)
    ws.bnorm2(bd, prec)
    ws.residual(prec, bd, x, r, r32)
    first = ws.read(with_cycle=False)
    if sqrt_in(prec, ws.bn2()) == 0.0:
        raise ZeroRightHandSideError("right-hand side is identically zero")
    baseline = sqrt_in(prec, first.rn2)
    history = [HistoryEntry(0, "outer", None, 1.0 if baseline else 0.0)]
    if baseline == 0.0:
        return ConvergenceReport(True, 0, 0, 0.0, history, False, x, baseline,
                                 phase_iters={"inner": 0, "outer": 0})
    floor = 10.0 * low.unit_roundoff
    rn2_low = first.rn2_low
    explicit = 1.0
    total = refinements = zero_streak = 0
    stalled = converged = False
    lib = D.lib()
    while True:
        if explicit <= cfg.rtol:
            converged = True
            break
        if refinements >= cfg.max_refinements:
            break
        remaining = cfg.inner.max_iters - total
        if remaining <= 0:
            break
        r_low_norm = sqrt_in(low, rn2_low)
        if r_low_norm == 0.0:
            refinements += 1
            zero_streak += 1
            if zero_streak >= 2:
                stalled = True
                break
            continue
        cap = max(1, min(cfg.inner.m, remaining))
        ws.cycle(low, r32, OFF_RN2_LOW, zeros32, u32, cap, floor, None, cfg.inner.breakdown_rule,
                 cfg.inner.orthogonalization, M)
        _lib.check(lib.mpk_ir_update(n, D.ptr(x), D.ptr(u32), ws.ws.at(OFF_CHANGED), D.stream()))
        ws.residual(prec, bd, x, r, r32)
        out = ws.read()
        for i, rel in enumerate(out.implicit):
            history.append(HistoryEntry(total + i + 1, "inner", rel * r_low_norm / baseline, None))
        total += out.steps
        refinements += 1
        zero_streak = 0 if out.changed else zero_streak + 1
        rn2_low = out.rn2_low
        explicit = sqrt_in(prec, out.rn2) / baseline
        history.append(HistoryEntry(total, "outer", None, explicit))
        if zero_streak >= 2:
            stalled = True
            break
    return ConvergenceReport(converged, total, refinements, explicit, history, False, x, baseline,
                             stalled=stalled, phase_iters={"inner": total, "outer": refinements})


# ---------------------------------------------------------------------------
# virtual ranks on one GPU (tests, single-GPU development boxes)
# ---------------------------------------------------------------------------

def run_virtual_ranks(nranks: int, fn):
    """Run fn(comm) for P virtual ranks, each in its own thread with its own
    CUDA stream on the current device; returns the per-rank results (or
    re-raises the first exception)."""
    t = D.torch()
    sh = _ThreadShared(nranks)
    dev = D.device()
    results = [None] * nranks
    errors = [None] * nranks

    def body(rank):
        try:
            t.cuda.set_device(dev)
            with t.cuda.stream(t.cuda.Stream(device=dev)):
                results[rank] = fn(ThreadComm(sh, rank))
                t.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errors[rank] = e
            sh.barrier.abort()

    threads = [threading.Thread(target=body, args=(q,)) for q in range(nranks)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for e in errors:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errors:
        if e is not None:
            raise e
    return results
