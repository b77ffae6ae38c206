"""The local-view jacobi_2d benchmark (paper §4.3 listing; the reference's
``sdfgkit.dist.benchmark`` API: JACOBI2D_LOCAL_VIEW, build_graph,
rank_bindings, run — pkg/tests/test_dist.py:9, 86-92, 288-306,
test_acceptance.py:17, 285-317).

Every rank of a Pr x Pc grid owns an lNx x lNy block of jacobi_2d's interior
plus a one-cell halo ring; each half step posts four sends and four receives
(north, south — rows; west, east — strided columns) and waits for them before
its 5-point update, so a step posts 8 sends per rank.  A rank on the global
boundary talks to PROC_NULL (-1) on that side: the post completes without
moving data and its halo keeps the global boundary values (comm.PROC_NULL).
The update is the global program's tasklet in the same op order, so the
result is bitwise equal to the shared-memory run.

The program text is JACOBI2D_LOCAL_VIEW (= programs/jacobi2d_local_view.dpy);
its graph was compiled by the reference frontend
(tests/golden/make_extra_graphs.py) and ships as jacobi2d_local_view.json
next to this module."""

from __future__ import annotations

import pathlib

import numpy as np

from .. import sdfg
from . import ProcessGrid, DistError

HERE = pathlib.Path(__file__).resolve().parent

JACOBI2D_LOCAL_VIEW = """\
def jacobi2d_local_view(TSTEPS: i32, A: f64[lNx + 2, lNy + 2], B: f64[lNx + 2, lNy + 2], nn: i32, ns: i32, nw: i32, ne: i32):
    req = requests(8)
    for t in range(1, TSTEPS):
        comm_isend(A[1, 1:lNy + 1], nn, 0, req[0])
        comm_isend(A[lNx, 1:lNy + 1], ns, 1, req[1])
        comm_isend(A[1:lNx + 1, 1], nw, 2, req[2])
        comm_isend(A[1:lNx + 1, lNy], ne, 3, req[3])
        comm_irecv(A[0, 1:lNy + 1], nn, 1, req[4])
        comm_irecv(A[lNx + 1, 1:lNy + 1], ns, 0, req[5])
        comm_irecv(A[1:lNx + 1, 0], nw, 3, req[6])
        comm_irecv(A[1:lNx + 1, lNy + 1], ne, 2, req[7])
        comm_waitall(req)
        for i, j in map[1:lNx + 1, 1:lNy + 1]:
            B[i, j] = 0.2 * (A[i, j] + A[i, j - 1] + A[i, j + 1] + A[i + 1, j] + A[i - 1, j])
        comm_isend(B[1, 1:lNy + 1], nn, 4, req[0])
        comm_isend(B[lNx, 1:lNy + 1], ns, 5, req[1])
        comm_isend(B[1:lNx + 1, 1], nw, 6, req[2])
        comm_isend(B[1:lNx + 1, lNy], ne, 7, req[3])
        comm_irecv(B[0, 1:lNy + 1], nn, 5, req[4])
        comm_irecv(B[lNx + 1, 1:lNy + 1], ns, 4, req[5])
        comm_irecv(B[1:lNx + 1, 0], nw, 7, req[6])
        comm_irecv(B[1:lNx + 1, lNy + 1], ne, 6, req[7])
        comm_waitall(req)
        for i, j in map[1:lNx + 1, 1:lNy + 1]:
            A[i, j] = 0.2 * (B[i, j] + B[i, j - 1] + B[i, j + 1] + B[i + 1, j] + B[i - 1, j])
"""


def build_graph() -> sdfg.Graph:
    """The compiled local-view program (schema v1, reference frontend)."""
    return sdfg.load(HERE / "jacobi2d_local_view.json")


def _dims(grid) -> tuple:
    dims = tuple(grid.dims if isinstance(grid, ProcessGrid) else grid)
    return dims if len(dims) == 2 else (dims[0], 1)


def rank_bindings(n: int, grid, tsteps: int | None = None) -> list:
    """Per-rank symbols of an n x n jacobi_2d on ``grid``: the block extents
    lNx x lNy of the (n - 2)^2 interior and the four neighbour ranks (-1 on
    the global boundary)."""
    pr, pc = _dims(grid)
    if (n - 2) % pr or (n - 2) % pc:
        raise DistError(f"the {n - 2} x {n - 2} interior does not divide over a {pr}x{pc} grid "
                        "(divisible block sizes required)")
    lnx, lny = (n - 2) // pr, (n - 2) // pc
    out = []
    for r in range(pr * pc):
        i, j = divmod(r, pc)
        b = {"lNx": lnx, "lNy": lny,
             "nn": (i - 1) * pc + j if i > 0 else -1,
             "ns": (i + 1) * pc + j if i < pr - 1 else -1,
             "nw": i * pc + j - 1 if j > 0 else -1,
             "ne": i * pc + j + 1 if j < pc - 1 else -1}
        if tsteps is not None:
            b["TSTEPS"] = tsteps
        out.append(b)
    return out


def windows(n: int, grid) -> list:
    """Per rank, the global (row, col) slices of its local arrays (interior
    block plus the halo ring)."""
    pr, pc = _dims(grid)
    lnx, lny = (n - 2) // pr, (n - 2) // pc
    return [(slice(i * lnx, i * lnx + lnx + 2), slice(j * lny, j * lny + lny + 2))
            for i in range(pr) for j in range(pc)]


def run(n: int, tsteps: int, grid, A, B, device: int = 0):
    """Run the benchmark on ``grid`` logical ranks on the B200 (simrun.RankSim:
    every rank a GpuExecutor, the messages through comm.RankComm).  Returns
    ({"A", "B"} global arrays assembled from the ranks' interior blocks,
    instr = {"per_rank": {r: counters}, "collective_ops": 0})."""
    from ..machine import ExecContext
    from ..simrun import RankSim

    dims = _dims(grid)
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    binds = rank_bindings(n, dims, tsteps)
    wins = windows(n, dims)
    stores = [{"A": A[w].copy(), "B": B[w].copy()} for w in wins]
    ctx = ExecContext(bindings={"TSTEPS": tsteps})
    sim = RankSim(build_graph(), dims, ctx, binds, stores=stores, device=device)
    try:
        _, instr = sim.run()
        outA, outB = A.copy(), B.copy()
        for r, (rs, cs) in enumerate(wins):
            st = sim.ranks[r].machine.store
            inner = (slice(rs.start + 1, rs.stop - 1), slice(cs.start + 1, cs.stop - 1))
            outA[inner] = np.asarray(st["A"])[1:-1, 1:-1]
            outB[inner] = np.asarray(st["B"])[1:-1, 1:-1]
    finally:
        sim.close()
    return {"A": outA, "B": outB}, instr


__all__ = ["JACOBI2D_LOCAL_VIEW", "build_graph", "rank_bindings", "windows", "run"]
