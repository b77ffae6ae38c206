"""CPU ORACLE — test infrastructure only: the reference's in-process rank
simulator (``sdfgkit.dist`` is absent from the mounted reference; its
contract is SPEC.md:505-603 and the tests pkg/tests/test_dist.py pins),
restated over ``interp_ref`` machines, numpy data, one host thread per
logical rank.

Semantics:
* root = rank 0 holds the global containers; other ranks get zero
  placeholders for non-transient inputs and skip nodes that touch only
  global (non DISTRIBUTED_LOCAL) containers (interp.py:199-206, 343-359);
* Scatter / Gather: 1-D blocks of the flattened (dense) view (529-530);
  BlockScatter / BlockGather: block layout of the node's ``dist`` grid, a
  1-D grid splitting the first dimension (532-534); uneven extents raise;
* Bcast from the root; Reduce (``comm`` REDUCE) combines the ranks'
  contributions with the node's operator, in rank order, into the root's
  output with the output memlet's WCR (531);
* DIST_MATMUL: C_local (=|+=) A @ B over the grid (SUMMA), computed here
  as the block product of the gathered panels (same blocks, same result);
* Isend snapshots its view, Irecv completes at Waitall, matching on
  (src, dst, tag) FIFO; an unmatched message is a DeadlockError.
Counters: messages_posted / delivered, comm_bytes (bytes sent + received),
collective_calls (every rank counts each collective it calls).
"""

from __future__ import annotations

import math
import threading

import numpy as np

from oracle import interp_ref as I
from paper_2107_00555_b200 import sdfg, symexpr

TIMEOUT = 30.0


class DeadlockError(RuntimeError):
    pass


class SimError(RuntimeError):
    pass


class _Hub:
    def __init__(self, P):
        self.P = P
        self.cv = threading.Condition()
        self.slots: dict = {}
        self.mail: dict = {}
        self.err = None

    def exchange(self, key, rank, value):
        """All ranks deposit under ``key``; returns {rank: value}."""
        with self.cv:
            self.slots.setdefault(key, {})[rank] = value
            self.cv.notify_all()
            ok = self.cv.wait_for(lambda: len(self.slots[key]) == self.P or self.err, TIMEOUT)
            if self.err:
                raise self.err
            if not ok:
                self.err = DeadlockError(f"collective {key} not reached by every rank")
                self.cv.notify_all()
                raise self.err
            return dict(self.slots[key])


def _owned(extent, griddim, coord, block):
    """Indices of one dim owned by ``coord``: blocks of ``block`` dealt
    round-robin (block = extent / griddim is the plain block layout)."""
    idx = []
    for start in range(coord * block, extent, griddim * block):
        idx.extend(range(start, min(start + block, extent)))
    return idx


def _blocks(gshape, gdims, coords, scheme="block", blocks=None):
    """np.ix_ index of the rank's part (block needs
    divisible extents, block-cyclic does not)."""
    gdims = list(gdims)
    while len(gdims) > len(gshape) and gdims[-1] == 1:
        gdims.pop()
    out = []
    for d, n in enumerate(gshape):
        if d < len(gdims):
            if scheme == "block":
                if n % gdims[d]:
                    raise SimError(f"extent {n} not covered by grid dim {gdims[d]} (divisible)")
                b = n // gdims[d]
            else:
                b = int(blocks[d]) if blocks else -(-n // gdims[d])
            out.append(_owned(n, gdims[d], coords[d], b))
        else:
            out.append(list(range(n)))
    return np.ix_(*out)


def _dist_of(n, env, gdims):
    a = n.attrs.get("dist") or {}
    dims = tuple(a.get("grid") or gdims)
    scheme = a.get("scheme", "block")
    blocks = None
    if scheme == "block_cyclic" and a.get("block"):
        blocks = [symexpr.evaluate(symexpr.parse(str(b)), env) for b in a["block"]]
    return dims, scheme, blocks


class RankMachine(I.Machine):
    def __init__(self, g, bindings, store, rank, P, grid_dims, hub, counters):
        super().__init__(g, bindings, store, {}, counters)
        self.rank, self.P, self.gdims, self.hub = rank, P, tuple(grid_dims), hub
        self.local = {n for n, c in g.containers.items() if c.storage == "distributed_local"}
        self.seq = 0
        self.pending = []
        self.msg_seq = 0

    def exec_node(self, st, n, env):
        if self.rank != 0 and self.local and self._root_only(st, n):
            return
        super().exec_node(st, n, env)

    def _root_only(self, st, n):
        if isinstance(n, sdfg.Library) and (n.kind in sdfg.COMM_KINDS or n.attrs.get("comm")):
            return False
        edges = st.in_edges(n) + st.out_edges(n)
        if isinstance(n, sdfg.MapEntry):
            ex = st.exit_of(n)
            edges = edges + st.in_edges(ex) + st.out_edges(ex)
        conts = {e.memlet.container for e in edges if e.memlet is not None}
        return bool(conts) and not (conts & self.local)

    # -- communication nodes ---------------------------------------------------

    def _ckey(self, kind):
        self.seq += 1
        return (kind, self.seq)

    def _coords(self, dims, r):
        return (r // dims[1], r % dims[1]) if len(dims) == 2 else (r,)

    def exec_library(self, st, n, env):
        if not (n.kind in sdfg.COMM_KINDS or n.attrs.get("comm")):
            return super().exec_library(st, n, env)
        C = self.counters
        ins = {e.dst_conn: e for e in st.in_edges(n) if e.memlet is not None}
        outs = {e.src_conn: e for e in st.out_edges(n) if e.memlet is not None}
        k = n.kind
        if k in ("isend", "irecv"):
            peer = int(symexpr.evaluate(n.attrs["peer"], env))
            tag = int(symexpr.evaluate(n.attrs["tag"], env))
            m = (ins if k == "isend" else outs)["buf"].memlet
            if peer == -1:  # MPI_PROC_NULL: posted, nothing moves
                C.messages_posted += k == "isend"
                return
            if k == "isend":
                data = np.array(self.read(m, env, st.label, n.id))
                self.pending.append(("s", peer, tag, data))
                C.messages_posted += 1
                C.comm_bytes += data.nbytes
            else:
                self.pending.append(("r", peer, tag, m, dict(env)))
            return
        if k == "waitall":
            sends = [(self.rank, x[1], x[2], x[3]) for x in self.pending if x[0] == "s"]
            allsends = self.hub.exchange(self._ckey("waitall"), self.rank, sends)
            box = {}
            for r in sorted(allsends):
                for src, dst, tag, data in allsends[r]:
                    box.setdefault((src, dst, tag), []).append(data)
            for x in self.pending:
                if x[0] != "r":
                    continue
                q = box.get((x[1], self.rank, x[2]))
                if not q:
                    raise DeadlockError(f"waitall pending: nothing sent {x[1]}->{self.rank} "
                                        f"tag {x[2]}")
                data = q.pop(0)
                ranges = symexpr.eval_subset(x[3].subset, x[4])
                self.write(x[3], data.reshape(tuple(len(r) for r in ranges)), x[4], st.label, n.id)
                C.messages_delivered += 1
                C.comm_bytes += data.nbytes
            self.pending = []
            return
        a_m = ins["a"].memlet
        o_e = outs["out"]
        C.collective_calls += 1
        if k in ("scatter", "block_scatter", "bcast"):
            g = np.array(self.read(a_m, env, st.label, n.id)) if self.rank == 0 else None
            parts = self.hub.exchange(self._ckey(k), self.rank, g)
            G = parts[0]
            if k == "bcast":
                v = G
            elif k == "scatter":
                flat = G.reshape(-1)
                if flat.size % self.P:
                    raise SimError("flat scatter: extent not divisible")
                c = flat.size // self.P
                v = flat[self.rank * c:(self.rank + 1) * c]
            else:
                dims, scheme, blocks = _dist_of(n, env, self.gdims)
                v = G[_blocks(G.shape, dims, self._coords(dims, self.rank), scheme, blocks)]
            ranges = symexpr.eval_subset(o_e.memlet.subset, env)
            self.write(o_e.memlet, np.asarray(v).reshape(tuple(len(r) for r in ranges)), env,
                       st.label, n.id)
            if self.P > 1:
                C.comm_bytes += np.asarray(v).nbytes
            return
        if k in ("gather", "block_gather"):
            loc = np.array(self.read(a_m, env, st.label, n.id))
            parts = self.hub.exchange(self._ckey(k), self.rank, loc)
            if self.rank == 0:
                gr = symexpr.eval_subset(o_e.memlet.subset, env)
                gshape = tuple(len(r) for r in gr)
                G = np.zeros(gshape)
                if k == "gather":
                    G = np.concatenate([parts[r].reshape(-1) for r in range(self.P)]).reshape(gshape)
                else:
                    dims, scheme, blocks = _dist_of(n, env, self.gdims)
                    for r in range(self.P):
                        sl = _blocks(gshape, dims, self._coords(dims, r), scheme, blocks)
                        G[sl] = parts[r].reshape(G[sl].shape)
                self.write(o_e.memlet, G, env, st.label, n.id)
            if self.P > 1:
                C.comm_bytes += loc.nbytes
            return
        if k == "reduce":
            loc = np.array(self.read(a_m, env, st.label, n.id), dtype=np.float64)
            parts = self.hub.exchange(self._ckey(k), self.rank, loc)
            fn = {"add": np.add, "mul": np.multiply, "min": np.minimum,
                  "max": np.maximum}[n.attrs.get("op", "add")]
            acc = parts[0].copy()
            for r in range(1, self.P):
                acc = fn(acc, parts[r])
            if self.rank == 0:
                ranges = symexpr.eval_subset(o_e.memlet.subset, env)
                self.write(o_e.memlet, acc.reshape(tuple(len(r) for r in ranges)), env, st.label,
                           n.id)
            return
        if k == "dist_matmul":
            la = np.array(self.read(ins["a"].memlet, env, st.label, n.id))
            lb = np.array(self.read(ins["b"].memlet, env, st.label, n.id))
            dims = tuple(n.attrs.get("dist", {}).get("grid") or self.gdims)
            if len(dims) == 1:
                dims = (dims[0], 1)
            Pr, Pc = dims
            parts = self.hub.exchange(self._ckey(k), self.rank, (la, lb))
            i, j = self._coords(dims, self.rank)
            A = np.concatenate([parts[i * Pc + jj][0] for jj in range(Pc)], axis=1)
            B = np.concatenate([parts[ii * Pc + j][1] for ii in range(Pr)], axis=0)
            ranges = symexpr.eval_subset(o_e.memlet.subset, env)
            self.write(o_e.memlet, (A @ B).reshape(tuple(len(r) for r in ranges)), env, st.label,
                       n.id)
            return
        raise SimError(f"collective '{k}' not supported")


def sim_run(g, grid_dims, bindings, store, rank_bindings=None, rank_stores=None,
            all_outputs=False):
    """(rank 0's outputs, per-rank counters) of ``g`` on P logical ranks
    (``rank_stores``: per-rank inputs of local-view programs; ``all_outputs``:
    every rank's outputs as a list)."""
    from paper_2107_00555_b200 import distribution as DI

    doc = g if isinstance(g, dict) else None
    g = sdfg.as_graph(g)
    doc = doc or g.doc or {}
    P = math.prod(grid_dims)
    hub = _Hub(P)
    ms, errs = [], [None] * P
    for r in range(P):
        b = DI.local_bindings(doc, grid_dims, dict(bindings), r)
        if rank_bindings is not None:
            b.update(rank_bindings[r])
        st = dict(rank_stores[r]) if rank_stores is not None else dict(store)
        if r and rank_stores is None:  # root-resident containers: placeholders
            for name, c in g.containers.items():
                if not c.transient and name not in st:
                    st[name] = np.zeros(tuple(symexpr.evaluate(d, b) for d in c.shape))
        c = I.Counters()
        for f in ("messages_posted", "messages_delivered", "comm_bytes", "collective_calls"):
            setattr(c, f, 0)
        ms.append(RankMachine(g, b, st, r, P, grid_dims, hub, c))

    def work(r):
        try:
            ms[r].run()
        except BaseException as ex:  # noqa: BLE001
            errs[r] = ex
            with hub.cv:
                hub.err = hub.err or ex
                hub.cv.notify_all()

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    e = next((x for x in errs if x is not None), None)
    if e is not None:
        raise e
    outs = [m.outputs() for m in ms] if all_outputs else ms[0].outputs()
    return outs, {r: dict(ms[r].counters.__dict__) for r in range(P)}
