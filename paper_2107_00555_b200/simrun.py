"""``sim_run`` / ``RankSim``: the reference's in-process multi-rank executor
(pkg/tests/test_dist.py:41-52, 124-141, 309-319),
restated on the B200.

P logical ranks of a distributed (global-view, distribute.py) or local-view
(explicit Isend / Irecv / Waitall) program run in ONE process on one device:
every rank is a ``GpuExecutor`` with its own HBM buffers and stream, driven
by its own host thread; its communication nodes go to the same
``comm.RankComm`` that drives NCCL in the one-process-per-GPU runner, with
the NCCL communicator replaced by ``HubComm`` — a mailbox of device buffers
matched on (source, destination) FIFO order, data moved by device-to-device
copies.  Before any rank launches anything, every rank walks its state
machine dry: collective sequences must agree (``CollectiveOrderError``) and
every message must be matched (``DeadlockError``), exactly the checks of the
NCCL runner.  Data movement is deterministic (fixed rank order in
reductions), so the rank scheduling order cannot change results
(``rank_order`` is accepted for the reference's signature: it fixes the
order in which ranks are created and their dry walks checked).

Root = rank 0 holds the global containers (``ctx.store``); the other ranks
get zero placeholders and skip root-resident ops (interp.py:199-206,
343-359).  Returns (rank 0's outputs, {"per_rank": {r: counters},
"collective_ops": collectives the program executed}).
"""

from __future__ import annotations

import threading

import numpy as np

from . import comm as C, distribution as DI, runtime as rt, sdfg

DeadlockError = C.DeadlockError
SimError = C.SimError
CollectiveOrderError = C.CollectiveOrderError
TIMEOUT_S = 60.0


class _Hub:
    def __init__(self, world: int):
        self.world = world
        self.cv = threading.Condition()
        self.mail: dict = {}  # (src, dst) -> list of [ptr, nbytes, consumed?]
        self.coll: dict = {}  # (kind, seq) -> {rank: (ptr, nbytes)}
        self.done: dict = {}  # (kind, seq) -> ranks finished reading
        self.error = None

    def wait(self, pred, what):
        if not self.cv.wait_for(lambda: pred() or self.error is not None, TIMEOUT_S):
            self.error = DeadlockError(f"rank simulator: {what} never completed")
        if self.error is not None:
            raise self.error


class HubComm:
    """NcclComm's interface (p2p / bcast / allreduce_f64 / close) between the
    logical ranks of one process."""

    def __init__(self, hub: _Hub, rank: int):
        self.hub, self.rank = hub, rank
        self.seq = {"bcast": 0, "allreduce": 0}

    def _sync(self, stream):
        rt.check(rt.lib().b2_stream_sync(stream), "sync")

    def p2p(self, ops, stream) -> int:
        hub, me = self.hub, self.rank
        self._sync(stream)  # the staged sends are complete
        mine = []
        with hub.cv:
            for send, peer, ptr, nbytes in ops:
                if send:
                    ent = [ptr, nbytes, False]
                    hub.mail.setdefault((me, peer), []).append(ent)
                    mine.append(ent)
            hub.cv.notify_all()
        sent = sum(n for s, _, _, n in ops if s)
        for send, peer, ptr, nbytes in ops:
            if send:
                continue
            with hub.cv:
                hub.wait(lambda: bool(hub.mail.get((peer, me))), f"receive {peer}->{me}")
                src_ptr, src_bytes, _ = ent = hub.mail[(peer, me)].pop(0)
            if src_bytes != nbytes:
                raise SimError(f"message {peer}->{me}: {src_bytes} bytes sent, {nbytes} expected")
            rt.check(rt.lib().b2_memcpy_d2d(ptr, src_ptr, nbytes, stream), "p2p copy")
            self._sync(stream)
            with hub.cv:
                ent[2] = True
                hub.cv.notify_all()
        with hub.cv:  # the staging buffers may be reused once consumed
            hub.wait(lambda: all(e[2] for e in mine), f"sends of rank {me} consumed")
        return sent

    def _collective(self, kind, ptr, nbytes, stream):
        hub, me = self.hub, self.rank
        self._sync(stream)
        key = (kind, self.seq[kind])
        self.seq[kind] += 1
        with hub.cv:
            hub.coll.setdefault(key, {})[me] = (ptr, nbytes)
            hub.cv.notify_all()
            hub.wait(lambda: len(hub.coll[key]) == hub.world, f"{kind} #{key[1]}")
            parts = dict(hub.coll[key])
        return key, parts

    def _finish(self, key):
        hub = self.hub
        with hub.cv:
            hub.done[key] = hub.done.get(key, 0) + 1
            hub.cv.notify_all()
            hub.wait(lambda: hub.done[key] == hub.world, f"{key[0]} #{key[1]} drain")

    def bcast(self, ptr: int, nbytes: int, root: int, stream) -> None:
        key, parts = self._collective("bcast", ptr, nbytes, stream)
        if self.rank != root:
            rt.check(rt.lib().b2_memcpy_d2d(ptr, parts[root][0], nbytes, stream), "bcast copy")
            self._sync(stream)
        self._finish(key)

    def allreduce_f64(self, ptr: int, count: int, wcr: str, stream) -> None:
        key, parts = self._collective("allreduce", ptr, 8 * count, stream)
        vals = []
        for r in range(self.hub.world):  # fixed rank order: deterministic
            a = np.empty(count, dtype=np.float64)
            rt.check(rt.lib().b2_memcpy_d2h(a.ctypes.data, parts[r][0], 8 * count, stream), "d2h")
            self._sync(stream)
            vals.append(a)
        self._finish(key)
        op = {"add": np.add, "mul": np.multiply, "min": np.minimum, "max": np.maximum}.get(wcr)
        if op is None:
            raise SimError(f"reduce operator '{wcr}' is not supported")
        acc = vals[0].copy()
        for v in vals[1:]:
            acc = op(acc, v)
        rt.check(rt.lib().b2_memcpy_h2d(ptr, acc.ctypes.data, 8 * count, stream), "h2d")
        self._sync(stream)

    def close(self):
        pass


class _Store:
    """Host view of one rank's containers (downloaded on access)."""

    def __init__(self, ex):
        self.ex = ex

    def __getitem__(self, name):
        if name not in self.ex.buf.ptr:
            raise KeyError(name)
        out = self.ex.download(name)
        self.ex.sync()
        return out

    def __contains__(self, name):
        return name in self.ex.buf.ptr


class _Machine:
    def __init__(self, ex, ctx):
        self.ex = ex
        self.ctx = ctx
        self.store = _Store(ex)


class _Rank:
    def __init__(self, rank, machine):
        self.rank = rank
        self.machine = machine


def _grid(grid):
    from .dist import ProcessGrid

    return grid if hasattr(grid, "dims") else ProcessGrid(grid)


class RankSim:
    """P logical ranks of ``g`` on one device (see module doc)."""

    def __init__(self, g, grid, ctx, bindings=None, rank_order=None, device: int = 0,
                 stores=None):
        from .machine import Counters, ExecContext, GpuExecutor, InterpOptions

        self.grid = _grid(grid)
        P = self.grid.size
        doc = g if isinstance(g, dict) else None
        self.g = sdfg.as_graph(g)
        doc = doc or self.g.doc or {}
        if bindings is not None and len(bindings) != P:
            raise SimError(f"{len(bindings)} rank bindings for {P} ranks")
        order = list(rank_order) if rank_order is not None else list(range(P))
        if sorted(order) != list(range(P)):
            raise SimError(f"rank order {order} is not a permutation of 0..{P - 1}")
        self.ctx = ctx
        self.stores = stores  # optional per-rank inputs (local-view programs)
        self.hub = _Hub(P)
        self.ranks = [None] * P
        self.comms = [None] * P
        for r in order:
            b = DI.local_bindings(doc, self.grid, dict(ctx.bindings), r)
            if bindings is not None:
                b.update(bindings[r])
            rc = C.RankComm(r, P, self.grid)
            ex = GpuExecutor(self.g, b, device=device, options=InterpOptions(), comm=rc)
            ex.capturable = False  # host-synchronous collectives: eager launches
            ex.device_branching = False
            rc.dry = True
            ex._instantiate_children()
            rc.dry = False
            rc.finish_dry()
            rctx = ExecContext(bindings=b, counters=Counters(), rank=r)
            self.ranks[r] = _Rank(r, _Machine(ex, rctx))
            self.comms[r] = rc
        for r in range(P):
            if self.comms[r].colls != self.comms[0].colls:
                raise CollectiveOrderError(
                    f"rank {r} calls collectives {self.comms[r].colls}, rank 0 "
                    f"{self.comms[0].colls}")
        for c in self.comms:
            c.raise_dry_errors()
        C.check_matching([c.records for c in self.comms])
        for r in range(P):
            self.comms[r].nccl = HubComm(self.hub, r)

    def _inputs(self, r):
        ex = self.ranks[r].machine.ex
        if self.stores is not None:
            return dict(self.stores[r])
        store = dict(getattr(self.ctx, "store", {}))
        if r == 0:
            return store
        out = {}
        for name, c in ex.g.containers.items():
            if c.transient:
                continue
            if name in store:
                out[name] = store[name]
            else:  # root-resident container: a placeholder this rank never reads
                out[name] = np.zeros(ex.buf.shape[name] if c.kind != "scalar" else ())
        return out

    def run(self):
        P = self.grid.size
        errors = [None] * P

        def work(r):
            m = self.ranks[r].machine
            try:
                store = self._inputs(r)
                keep = m.ex.prepare_inputs(store)
                m.ex.run_device(first_call=True, counters=m.ctx.counters)
                m.ex.sync()
                m.ex.check_flag()
                del keep
            except BaseException as exn:  # noqa: BLE001 - reported below
                errors[r] = exn
                with self.hub.cv:
                    if self.hub.error is None:
                        self.hub.error = exn if isinstance(exn, (DeadlockError, SimError)) else \
                            SimError(f"rank {r} failed: {exn}")
                    self.hub.cv.notify_all()

        threads = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(P)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        first = next((e for e in errors if e is not None), None)
        if first is not None:
            raise first
        out = self.ranks[0].machine.ex.outputs()
        per = {r: self.ranks[r].machine.ctx.counters.as_dict() for r in range(P)}
        # collective operations of the program (every rank takes part in
        # each; the root's count), as the reference's instrumentation
        return out, {"per_rank": per, "collective_ops": per[0]["collective_calls"]}

    def close(self):
        for rk, rc in zip(self.ranks, self.comms):
            rk.machine.ex.close()
            rc.close()


def sim_run(g, grid, ctx, bindings=None, rank_order=None):
    """The reference's ``sim_run(g, grid, ctx, bindings=None,
    rank_order=None) -> (outputs, instr)`` on one B200."""
    sim = RankSim(g, grid, ctx, bindings, rank_order)
    try:
        return sim.run()
    finally:
        sim.close()
