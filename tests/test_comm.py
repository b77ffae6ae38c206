"""Local-view message passing (comm.py): the cross-rank message-key check on
CPU, and the GPU runner on one rank (self-addressed messages, no-comm
decompositions).  Multi-rank transfers are NCCL grouped send/recv — the same
libb2 path the slab runner uses."""

import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN


def test_check_matching_fifo_per_key():
    from paper_2107_00555_b200.comm import check_matching

    # rank 0 sends tags 7 then 8 to rank 1; rank 1 posts the receives in the
    # opposite order: (src, dst, tag) matching still pairs them
    r0 = [[(True, 1, 7, 32), (True, 1, 8, 16), (False, 1, 9, 8)]]
    r1 = [[(False, 0, 8, 16), (False, 0, 7, 32), (True, 0, 9, 8)]]
    check_matching([r0, r1])
    check_matching([[[]], [[]]])  # waitall on empty requests: no-op


def test_check_matching_diagnostics():
    from paper_2107_00555_b200.comm import DeadlockError, check_matching

    with pytest.raises(DeadlockError, match="unmatched message"):
        check_matching([[[(True, 1, 3, 16)]], [[]]])
    with pytest.raises(DeadlockError, match="waitall pending"):
        check_matching([[[]], [[(False, 0, 3, 16)]]])
    with pytest.raises(DeadlockError, match="unmatched message"):  # size mismatch
        check_matching([[[(True, 1, 3, 16)]], [[(False, 0, 3, 8)]]])
    with pytest.raises(DeadlockError, match="outside"):
        check_matching([[[(True, 5, 3, 16)]]])
    # a receive posted one waitall later than its send does not match
    with pytest.raises(DeadlockError):
        check_matching([[[(True, 1, 1, 8)], []], [[], [(False, 0, 1, 8)]]])


@pytest.fixture(scope="module")
def pg():
    import torch.distributed as tdist

    if not tdist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        tdist.init_process_group("gloo", rank=0, world_size=1)
    yield


@pytest.mark.gpu
def test_halo_pair_self_exchange(pg):
    """pkg/tests/test_dist.py:121-140 on one rank addressing itself: the
    received column equals the sent one, byte and message counters match."""
    from paper_2107_00555_b200 import ExecContext, sdfg
    from paper_2107_00555_b200.comm import local_view_run

    g = sdfg.load(GOLDEN / "graphs" / "halo_pair.raw.json")
    lnx, lny = 4, 5
    rng = np.random.default_rng(2)
    A = rng.uniform(-1, 1, (lnx + 2, lny + 2))
    ctx = ExecContext(bindings={"lNx": lnx, "lNy": lny}).bind_inputs({"A": A})
    out, instr = local_view_run(g, ctx, [{"peer": 0, "me": 0}])
    i, j = np.meshgrid(np.arange(lnx + 2), np.arange(lny + 2), indexing="ij")
    buf = 0 * 100.0 + i * 10.0 + j + A
    ref = np.zeros_like(A)
    ref[1:-1, -1] = buf[1:-1, -2]
    assert np.array_equal(out["A"], ref)
    c = instr["per_rank"][0]
    assert c["comm_bytes"] == 2 * lnx * 8
    assert c["messages_posted"] == 1 and c["messages_delivered"] == 1


@pytest.mark.gpu
def test_overlapping_receives_race(pg):
    from paper_2107_00555_b200 import ExecContext, sdfg
    from paper_2107_00555_b200.comm import SimError, local_view_run

    g = sdfg.load(GOLDEN / "graphs" / "overlap_recv.raw.json")
    ctx = ExecContext(bindings={"lNx": 2, "lNy": 2}).bind_inputs({"A": np.zeros((4, 4))})
    with pytest.raises(SimError, match="overlapping"):
        local_view_run(g, ctx, [{"peer": 0}])


@pytest.mark.gpu
@pytest.mark.parametrize("N,T", [(12, 4), (33, 5)])
def test_jacobi2d_local_single_rank_equals_global(pg, N, T):
    """The local-view jacobi_2d on a 1-rank decomposition (no neighbours: the
    halo rows are the global boundary) is bitwise the corpus jacobi_2d."""
    from oracle import kernels_np as K
    from paper_2107_00555_b200 import ExecContext, sdfg
    from paper_2107_00555_b200.comm import local_view_run

    g = sdfg.load(GOLDEN / "graphs" / "jacobi2d_local.raw.json")
    rng = np.random.default_rng(N)
    A = rng.uniform(-1, 1, (N, N))
    B = rng.uniform(-1, 1, (N, N))
    ctx = ExecContext(bindings={"lNx": N - 2, "N": N, "TSTEPS": T}).bind_inputs(
        {"A": A.copy(), "B": B.copy()})
    out, instr = local_view_run(g, ctx, [{"up": -1, "down": -1}])
    K.jacobi_2d(A, B, T)
    assert np.array_equal(out["A"], A) and np.array_equal(out["B"], B)
    assert instr["per_rank"][0]["messages_posted"] == 0


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_jacobi2d_rank_setup(P):
    """Row windows of the local-view decomposition: owned interior rows tile
    1..N-2 exactly, neighbours are adjacent ranks, edges have none."""
    from paper_2107_00555_b200.comm import jacobi2d_rank_setup

    N = 2 + 24 * 7
    owned = []
    for r in range(P):
        b, (lo, hi) = jacobi2d_rank_setup(N, P, r)
        assert hi - lo == b["lNx"] + 2
        owned += list(range(lo + 1, hi - 1))
        assert b["up"] == (r - 1 if r else -1) and b["down"] == (r + 1 if r < P - 1 else -1)
    assert owned == list(range(1, N - 1))


def test_block_layout_spec_examples():
    """BlockScatter f64[4,4] over a 2x2 grid gives rank (0,1)
    rows 0-1, cols 2-3; uneven extents are an error; a 1-D grid splits the
    first dimension."""
    from paper_2107_00555_b200.comm import SimError, block_layout
    from paper_2107_00555_b200.dist import ProcessGrid

    g = ProcessGrid((2, 2))
    assert block_layout((4, 4), g.dims, g.coords(1)) == [(0, 2), (2, 2)]
    assert block_layout((8, 3), (4,), (3,)) == [(6, 2), (0, 3)]
    with pytest.raises(SimError, match="not covered"):
        block_layout((5, 4), (2, 2), (0, 0))


@pytest.mark.gpu
def test_block_scatter_gather_roundtrip_single_rank(pg):
    """BlockGather(map(BlockScatter(A))) on a 1x1 grid: local copies only."""
    from paper_2107_00555_b200 import ExecContext, sdfg
    from paper_2107_00555_b200.comm import local_view_run
    from paper_2107_00555_b200.dist import ProcessGrid

    g = sdfg.load(GOLDEN / "graphs" / "block_roundtrip.raw.json")
    rng = np.random.default_rng(4)
    A = rng.uniform(-1, 1, (6, 10))
    ctx = ExecContext(bindings={"N": 6, "M": 10, "lN": 6, "lM": 10}).bind_inputs(
        {"A": A, "B": np.zeros_like(A), "L": np.zeros_like(A)})
    out, instr = local_view_run(g, ctx, [{}], grid=ProcessGrid((1, 1)))
    assert np.array_equal(out["B"], A * 2.0 + 1.0)
    assert instr["collective_ops"] == 2 and instr["per_rank"][0]["comm_bytes"] == 0


def _doc(name):
    import json

    return json.loads((GOLDEN / "graphs" / f"{name}.json").read_text())


@pytest.mark.gpu
def test_flat_scatter_gather_bcast_reduce_single_rank(pg):
    """SCATTER / GATHER (1-D blocks of the flattened container), BCAST and
    REDUCE through the local-view runner on one rank: local
    copies, and the collective-call counter."""
    import json

    from paper_2107_00555_b200 import ExecContext, sdfg
    from paper_2107_00555_b200.comm import local_view_run

    d = _doc("block_roundtrip.raw")
    for st in d["states"]:
        for n in st["nodes"]:
            if n.get("type") == "library":
                n["kind"] = {"block_scatter": "scatter", "block_gather": "gather"}[n["kind"]]
    g = sdfg.loads(json.dumps(d))
    rng = np.random.default_rng(8)
    A = rng.uniform(-1, 1, (4, 6))
    ctx = ExecContext(bindings={"N": 4, "M": 6, "lN": 4, "lM": 6}).bind_inputs(
        {"A": A, "B": np.zeros_like(A), "L": np.zeros_like(A)})
    out, instr = local_view_run(g, ctx, [{}])
    assert np.array_equal(out["B"], A * 2.0 + 1.0) and instr["collective_ops"] == 2

    # bcast of the root's A into L, then reduce of L into B (sum over ranks)
    d2 = _doc("block_roundtrip.raw")
    d2["states"][0]["nodes"][0]["kind"] = "bcast"
    d2["states"][2]["nodes"][0]["kind"] = "reduce"
    # a collective reduce is a REDUCE library node marked "comm" (interp.py:444)
    d2["states"][2]["nodes"][0]["attrs"] = {"op": "add", "comm": True}
    g2 = sdfg.loads(json.dumps(d2))
    ctx2 = ExecContext(bindings={"N": 4, "M": 6, "lN": 4, "lM": 6}).bind_inputs(
        {"A": A, "B": np.zeros_like(A), "L": np.zeros_like(A)})
    out2, instr2 = local_view_run(g2, ctx2, [{}])
    assert np.array_equal(out2["B"], A * 2.0 + 1.0) and instr2["collective_ops"] == 2


@pytest.mark.parametrize("dims", [(2, 1), (1, 2), (2, 2), (4, 2), (2, 3), (3, 2)])
def test_summa_panel_ops_match_across_ranks(dims):
    """DIST_MATMUL's per-panel NCCL group (comm.summa_panel_ops): for every
    panel each receive has exactly one matching send (same bytes, A panels
    inside a grid row, B panels inside a grid column), and the owners of
    A's / B's panel l hold local panel la / lb of their blocks."""
    import math

    from paper_2107_00555_b200.comm import summa_panel_ops

    Pr, Pc = dims
    L = math.lcm(Pr, Pc)
    for l in range(L):
        sends, recvs = [], []
        owners_a, owners_b = set(), set()
        for r in range(Pr * Pc):
            i, j = divmod(r, Pc)
            ca, la, rb, lb, ops = summa_panel_ops(Pr, Pc, i, j, l, "A", 8, "B", 16)
            assert ca * (L // Pc) + la == l and rb * (L // Pr) + lb == l
            if j == ca:
                owners_a.add((i, j))
            if i == rb:
                owners_b.add((i, j))
            for send, peer, buf, nb in ops:
                pi, pj = divmod(peer, Pc)
                assert (pi == i) if buf == "A" else (pj == j)
                (sends if send else recvs).append((r, peer, buf, nb) if send else (peer, r, buf, nb))
        assert sorted(sends) == sorted(recvs)
        assert len(owners_a) == Pr and len(owners_b) == Pc
        assert len(recvs) == Pr * (Pc - 1) + Pc * (Pr - 1)


@pytest.mark.gpu
def test_dist_matmul_single_rank_is_local_matmul(pg):
    """A DIST_MATMUL node on a 1x1 grid degenerates to the
    local MATMUL with zero messages; K cut into one panel."""
    import json

    from paper_2107_00555_b200 import ExecContext, sdfg
    from paper_2107_00555_b200.comm import local_view_run

    d = _doc("matmul.raw")
    for st in d["states"]:
        for n in st["nodes"]:
            if n.get("type") == "library":
                n["kind"] = "dist_matmul"
                n["attrs"] = {"dist": {"grid": [1, 1], "scheme": "block"}}
    g = sdfg.loads(json.dumps(d))
    rng = np.random.default_rng(12)
    A, B = rng.uniform(-1, 1, (96, 160)), rng.uniform(-1, 1, (160, 72))
    ctx = ExecContext(bindings={"M": 96, "K": 160, "N": 72}).bind_inputs(
        {"A": A, "B": B, "C": np.full((96, 72), 7.0)})
    out, instr = local_view_run(g, ctx, [{}])
    ref = A @ B
    assert np.linalg.norm(out["C"] - ref) / np.linalg.norm(ref) <= 1e-12
    assert instr["collective_ops"] == 0 and instr["per_rank"][0]["comm_bytes"] == 0


@pytest.mark.parametrize("dims", [(2, 1), (1, 2), (2, 2), (2, 3), (4, 2)])
def test_summa_dataflow_emulated(dims):
    """The DIST_MATMUL data flow of comm.RankComm._dist_matmul replayed on
    the host: owners slice panel la / lb out of their local blocks, the
    summa_panel_ops groups deliver them, every rank accumulates PA @ PB —
    the assembled C equals A @ B."""
    import math

    from paper_2107_00555_b200.comm import summa_panel_ops

    Pr, Pc = dims
    L = math.lcm(Pr, Pc)
    M, N, K = 6 * Pr, 5 * Pc, 4 * L
    rng = np.random.default_rng(Pr * 10 + Pc)
    A, B = rng.uniform(-1, 1, (M, K)), rng.uniform(-1, 1, (K, N))
    am, ak, bk, bn, kb = M // Pr, K // Pc, K // Pr, N // Pc, K // L
    Ab = {(i, j): A[i * am:(i + 1) * am, j * ak:(j + 1) * ak] for i in range(Pr) for j in range(Pc)}
    Bb = {(i, j): B[i * bk:(i + 1) * bk, j * bn:(j + 1) * bn] for i in range(Pr) for j in range(Pc)}
    C = {(i, j): np.zeros((am, bn)) for i in range(Pr) for j in range(Pc)}
    for l in range(L):
        pa, pb, plan = {}, {}, {}
        for r in range(Pr * Pc):
            i, j = divmod(r, Pc)
            ca, la, rb, lb, ops = summa_panel_ops(Pr, Pc, i, j, l, "A", 0, "B", 0)
            plan[r] = ops
            if j == ca:
                pa[r] = Ab[(i, j)][:, la * kb:(la + 1) * kb]
            if i == rb:
                pb[r] = Bb[(i, j)][lb * kb:(lb + 1) * kb, :]
        for r, ops in plan.items():
            for send, peer, buf, _ in ops:
                if not send:
                    (pa if buf == "A" else pb)[r] = (pa if buf == "A" else pb)[peer]
        for r in range(Pr * Pc):
            C[divmod(r, Pc)] += pa[r] @ pb[r]
    full = np.block([[C[(i, j)] for j in range(Pc)] for i in range(Pr)])
    assert np.allclose(full, A @ B, rtol=1e-12, atol=1e-12)
