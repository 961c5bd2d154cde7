"""PFASST with ISDC sweeps (NEXT f4b; reading R33): the time-parallel driver.

PAPER.md P:207-209: PFASST "performs SDC sweeps on multiple levels combined with a forward transfer
of updated initial values in a manner similar to Parareal ... on each time level, only a single SDC
sweep is performed".  A block of P time slices (slice p = time step step0 + p) is iterated; every
slice is a two-level MLSDC handle (R32) whose per-slice phases run in the CUDA library
(include/isdc.h, ``isdc_pfasst_*``).  This module only schedules them and moves the dense end values
between slices: it computes nothing itself.

The algorithm is written ONCE, as the program of one slice (``slice_program``), a generator that
yields its communication requests:

    ("send", dst, tensor)   forward transfer to slice dst = p + 1 (non-blocking)
    ("recv", src, kind)     -> the next value sent by slice src = p - 1 (FIFO per pair); kind
                               "fine" (n^d) or "coarse" (n_c^d) -- the R33 order fixes it
    ("allmax", x)           -> max of x over all slices (the block's stop test)

Two transports run it:
* ``run_block_local``: all P slices in one process on one GPU (or, in the tests, on the CPU
  oracle's slice phases), the generators stepped round-robin with in-memory FIFOs;
* ``run_block_dist``: one slice per rank of a torch.distributed group (NCCL over NVLink between
  GPUs, gloo in the CPU tests): isend/irecv of the end values, all_reduce(MAX) of the residual.

Because every slice only reads what R33's dependencies give it, both transports compute the same
bits as the oracle's serial emulation (oracle/isdc_oracle.c ora_pfasst_block).

Order of the per-slice program (R33):
  predictor: residual of the spread state, injection + FAS; stages s = 0..p: (s >= 1: coarse node
             0 <- slice p-1's stage s-1 end value) coarse sweeps, send the coarse end to p+1;
             interpolate.
  iteration: send the fine end value to p+1; (p >= 1: fine node 0 <- the received value); fine
             sweep + residual; stop test on the max over slices; injection + FAS; (p >= 1: coarse
             node 0 <- slice p-1's coarse end value of this iteration) coarse sweeps; send the
             coarse end to p+1; interpolate.
"""
from __future__ import annotations

import collections
from dataclasses import dataclass, field
from typing import Callable, List, Optional


@dataclass
class SliceResult:
    iterations: int = 0
    converged: bool = False
    res_hist: List[float] = field(default_factory=list)      # this slice's residual per iteration
    block_hist: List[float] = field(default_factory=list)    # max over slices per iteration
    vcycles: int = 0
    coarse_vcycles: int = 0
    sent: int = 0          # bytes this slice sent forward
    recv: int = 0


class CudaSlice:
    """One PFASST slice on the CUDA path: an ``ISDC`` handle with mlsdc_levels = 2 (R32/R33)."""

    def __init__(self, handle, u0, step_index: int):
        if handle.p.mlsdc_levels != 2:
            raise ValueError("a PFASST slice needs an MLSDC handle (mlsdc_levels = 2)")
        self.h = handle
        self.h.set_initial(u0, step_index)
        self.vcycles = 0
        self.coarse_vcycles = 0
        self._end = None
        self.fine_shape = (handle.n,) * handle.dim
        self.coarse_shape = (handle.coarse_n(),) * handle.dim
        self.wants_torch = True

    def predict_restrict(self):
        self.h.pfasst_restrict()

    def fine(self) -> float:
        per, mx, cyc = self.h.sweep()
        self.vcycles += int(sum(cyc))
        self._end = None
        return mx

    def restrict(self):
        self.h.pfasst_restrict()

    def coarse(self, U0=None):
        Uend, cv = self.h.pfasst_coarse(U0)
        self.coarse_vcycles += cv
        return Uend

    def interpolate(self):
        self._end = self.h.pfasst_interpolate()
        return self._end

    def set_u0(self, u0):
        self.h.pfasst_set_u0(u0)
        self._end = None

    def end(self):
        return self.h.solution(-1)


def slice_program(p: int, P: int, sl, *, max_iters: int, fixed_iters: int = 0, tol: float = 1e-10,
                  predictor: bool = True, nbytes: Optional[Callable] = None):
    """The PFASST program of slice p of P (R33), as a generator of communication requests; returns a
    SliceResult.  ``sl`` provides the slice phases (CudaSlice, or the oracle's slice in the tests)."""
    res = SliceResult()
    size = nbytes or (lambda t: 0)
    if predictor:
        sl.predict_restrict()
        for s in range(p + 1):
            U0 = None
            if s >= 1:
                U0 = yield ("recv", p - 1, "coarse")
                res.recv += size(U0)
            Uend = sl.coarse(U0)
            if p + 1 < P:
                yield ("send", p + 1, Uend)
                res.sent += size(Uend)
        E = sl.interpolate()
    else:
        E = sl.end()
    kmax = fixed_iters if fixed_iters > 0 else max_iters
    k = 0
    while k < kmax:
        if p + 1 < P:
            yield ("send", p + 1, E)
            res.sent += size(E)
        if p >= 1:
            u0 = yield ("recv", p - 1, "fine")
            res.recv += size(u0)
            sl.set_u0(u0)
        r = sl.fine()
        k += 1
        rmax = yield ("allmax", r)
        res.res_hist.append(r)
        res.block_hist.append(rmax)
        if fixed_iters <= 0 and rmax < tol:
            res.converged = True
            break
        if k >= kmax:
            break
        sl.restrict()
        U0 = None
        if p >= 1:
            U0 = yield ("recv", p - 1, "coarse")
            res.recv += size(U0)
        Uend = sl.coarse(U0)
        if p + 1 < P:
            yield ("send", p + 1, Uend)
            res.sent += size(Uend)
        E = sl.interpolate()
    if fixed_iters > 0:
        res.converged = True
    res.iterations = k
    res.vcycles, res.coarse_vcycles = sl.vcycles, sl.coarse_vcycles
    return res


def run_block_local(slices, **kw) -> List[SliceResult]:
    """All slices of a block in this process: the slice programs stepped round-robin, messages in
    per-pair FIFOs, the stop test's max taken when every live slice has reached it."""
    P = len(slices)
    progs = [slice_program(p, P, slices[p], **kw) for p in range(P)]
    box = collections.defaultdict(collections.deque)     # (src, dst) -> values
    pending = [None] * P          # request a slice is blocked on
    reply = [None] * P            # value to send into the generator at its next resume
    done: List[Optional[SliceResult]] = [None] * P
    started = [False] * P
    while any(d is None for d in done):
        progressed = False
        for p in range(P):
            while done[p] is None:
                req = pending[p]
                if req is not None:
                    if req[0] == "recv":
                        q = box[(req[1], p)]
                        if not q:
                            break
                        reply[p], pending[p] = q.popleft(), None
                    elif req[0] == "allmax":
                        break      # resolved below once every live slice waits on it
                try:
                    if not started[p]:
                        started[p] = True
                        req = next(progs[p])
                    else:
                        req = progs[p].send(reply[p])
                except StopIteration as e:
                    done[p] = e.value
                    progressed = True
                    break
                reply[p] = None
                progressed = True
                if req[0] == "send":
                    box[(p, req[1])].append(req[2])
                    continue
                pending[p] = req
        live = [p for p in range(P) if done[p] is None]
        if live and all(pending[p] is not None and pending[p][0] == "allmax" for p in live):
            m = max(pending[p][1] for p in live)
            for p in live:
                reply[p], pending[p] = m, None
            progressed = True
        if not progressed:
            raise RuntimeError("PFASST local schedule deadlocked (a slice waits on a value never sent)")
    return done


def run_block_dist(sl, *, group=None, device=None, **kw) -> SliceResult:
    """This rank's slice of a block, one slice per rank of the torch.distributed group (slice p =
    rank p, P = world size): isend/irecv of the dense end values to the neighbours and an
    all_reduce(MAX) for the stop test.  ``device``: where the transport's tensors live -- the rank's
    GPU for NCCL (NVLink), None = host memory for gloo (CUDA slices then stage through the host)."""
    import torch
    import torch.distributed as dist

    p, P = dist.get_rank(group), dist.get_world_size(group)
    prog = slice_program(p, P, sl, **kw)
    sends = []
    reply = None
    first = True

    def as_tensor(x):
        return x if isinstance(x, torch.Tensor) else torch.from_numpy(x)

    while True:
        try:
            req = next(prog) if first else prog.send(reply)
        except StopIteration as e:
            for w, _ in sends:
                w.wait()
            return e.value
        first, reply = False, None
        if req[0] == "send":
            # the transport's device (CPU for gloo, the rank's GPU for NCCL); a copy, since the
            # slice may overwrite its buffer while the send is in flight
            t = as_tensor(req[2]).to(device if device is not None else torch.device("cpu")).contiguous().clone()
            sends.append((dist.isend(t, req[1], group=group), t))
        elif req[0] == "recv":
            reply = _recv(req[1], req[2], sl, device, group)
        else:
            dev = device if device is not None else torch.device("cpu")
            t = torch.tensor([float(req[1])], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            reply = float(t.item())


def _recv(src, kind, sl, device, group):
    """Blocking receive of the next end value from slice src, shaped by its kind."""
    import torch
    import torch.distributed as dist

    shape = sl.fine_shape if kind == "fine" else sl.coarse_shape
    dev = device if device is not None else torch.device("cpu")
    t = torch.empty(shape, dtype=torch.float64, device=dev)
    dist.recv(t, src, group=group)
    return t if getattr(sl, "wants_torch", True) else t.numpy()
