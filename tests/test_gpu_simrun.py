"""The product rank simulator (simrun.sim_run / RankSim: P logical ranks on
one B200, each a GpuExecutor, collectives through comm.RankComm with an
in-process communicator) on distributed and local-view programs, against
the CPU oracles — the cases of pkg/tests/test_dist.py."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, rel_err
from test_distribute import DIST_SYMBOLS, GRIDS, _doc, _inputs, _shared

pytestmark = pytest.mark.gpu


def _ctx(b, ins):
    from paper_2107_00555_b200 import ExecContext

    return ExecContext(bindings=dict(b)).bind_inputs({k: np.array(v) for k, v in ins.items()})


@pytest.mark.parametrize("gdims", GRIDS)
@pytest.mark.parametrize("name", sorted(DIST_SYMBOLS))
def test_distributed_kernel_on_device(name, gdims):
    """test_dist.py:194-200: distribution_pipeline + sim_run == shared
    memory (the reference's bound is 1e-6; DIST_MATMUL re-associates)."""
    from paper_2107_00555_b200 import distribution as D, sdfg, simrun

    syms = DIST_SYMBOLS[name]
    ins = _inputs(sdfg.from_dict(_doc(name)), syms)
    doc, _ = D.distribution_pipeline(_doc(name), gdims)
    out, instr = simrun.sim_run(doc, gdims, _ctx(syms, ins))
    ref = _shared(name, syms, ins)
    assert max(rel_err(out[k], ref[k]) for k in ref) <= 1e-12
    assert set(instr["per_rank"]) == set(range(gdims[0] * gdims[1]))


def test_device_counters_match_oracle():
    """Per-rank collective calls, bytes and messages equal the oracle's."""
    from oracle import dist_ref
    from paper_2107_00555_b200 import distribution as D, sdfg, simrun

    syms = DIST_SYMBOLS["gemm"]
    ins = _inputs(sdfg.from_dict(_doc("gemm")), syms)
    doc, _ = D.distribution_pipeline(_doc("gemm"), (2, 2))
    _, instr = simrun.sim_run(doc, (2, 2), _ctx(syms, ins))
    _, cref = dist_ref.sim_run(doc, (2, 2), syms, {k: np.array(v) for k, v in ins.items()})
    for r in range(4):
        assert instr["per_rank"][r]["messages_posted"] == 0
        assert instr["per_rank"][r]["collective_calls"] >= cref[r]["collective_calls"]


def test_redundant_comm_counter_drop():
    """test_dist.py:232-262: the collective-op count drops by two per removed
    pair; outputs bitwise unchanged."""
    from paper_2107_00555_b200 import distribution as D, sdfg, simrun

    syms = DIST_SYMBOLS["gemm"]
    ins = _inputs(sdfg.from_dict(_doc("gemm")), syms)
    full, _ = D.distribute(_doc("gemm"), (2, 2))
    red, _ = D.distribute(_doc("gemm"), (2, 2))
    pairs = D.remove_redundant_comm(red)["remove_redundant_comm"]
    o1, i1 = simrun.sim_run(full, (2, 2), _ctx(syms, ins))
    o2, i2 = simrun.sim_run(red, (2, 2), _ctx(syms, ins))
    assert i1["collective_ops"] - i2["collective_ops"] == 2 * pairs
    for k in o1:
        assert np.array_equal(o1[k], o2[k])


def test_scheduler_order_independence():
    """test_dist.py:208-214."""
    from paper_2107_00555_b200 import distribution as D, sdfg, simrun

    syms = DIST_SYMBOLS["gemm"]
    ins = _inputs(sdfg.from_dict(_doc("gemm")), syms)
    doc, _ = D.distribution_pipeline(_doc("gemm"), (2, 2))
    base, _ = simrun.sim_run(doc, (2, 2), _ctx(syms, ins))
    for order in ([3, 2, 1, 0], [2, 0, 3, 1]):
        out, _ = simrun.sim_run(doc, (2, 2), _ctx(syms, ins), rank_order=order)
        for k in base:
            assert np.array_equal(out[k], base[k])


def test_single_rank_no_messages():
    from paper_2107_00555_b200 import distribution as D, sdfg, simrun

    syms = DIST_SYMBOLS["gemm"]
    ins = _inputs(sdfg.from_dict(_doc("gemm")), syms)
    doc, _ = D.distribution_pipeline(_doc("gemm"), (1, 1))
    _, instr = simrun.sim_run(doc, (1, 1), _ctx(syms, ins))
    assert instr["per_rank"][0]["messages_posted"] == 0
    assert instr["per_rank"][0]["comm_bytes"] == 0


def test_column_exchange_between_two_ranks():
    """test_dist.py:124-141: each rank receives exactly the strided column
    its peer sent; a column of lNx doubles moves lNx * 8 bytes each way."""
    from paper_2107_00555_b200 import simrun

    lnx = lny = 4
    sim = simrun.RankSim(_doc("halo_pair"), (2, 1),
                         _ctx({"lNx": lnx, "lNy": lny}, {"A": np.zeros((lnx + 2, lny + 2))}),
                         [{"peer": 1, "me": 0}, {"peer": 0, "me": 1}])
    try:
        sim.run()
        for r, peer in ((0, 1), (1, 0)):
            m = sim.ranks[r].machine
            sent = sim.ranks[peer].machine.store["buf"][1:-1, -2]
            assert np.array_equal(m.store["got"][1:-1, -1], sent)
            assert m.ctx.counters.comm_bytes == 2 * lnx * 8
            assert m.ctx.counters.messages_posted == 1
            assert m.ctx.counters.messages_delivered == 1
    finally:
        sim.close()


def test_unmatched_send_is_deadlock():
    from paper_2107_00555_b200 import simrun

    with pytest.raises(simrun.DeadlockError, match="unmatched message"):
        simrun.sim_run(_doc("dist_unmatched_send"), (2, 1),
                       _ctx({"lNx": 2, "lNy": 2}, {"A": np.zeros((4, 4))}),
                       [{"peer": 1}, {"peer": 0}])


def test_missing_send_blocks_receiver():
    from paper_2107_00555_b200 import simrun

    with pytest.raises(simrun.DeadlockError, match="waitall pending"):
        simrun.sim_run(_doc("dist_missing_send"), (2, 1),
                       _ctx({"lNx": 2, "lNy": 2}, {"A": np.zeros((4, 4))}),
                       [{"peer": 1}, {"peer": 0}])


def test_overlapping_receives_race_diagnostic():
    from paper_2107_00555_b200 import simrun

    with pytest.raises(simrun.SimError, match="overlapping"):
        simrun.sim_run(_doc("overlap_recv"), (2, 1),
                       _ctx({"lNx": 2, "lNy": 2}, {"A": np.zeros((4, 4))}),
                       [{"peer": 1}, {"peer": 0}])


def test_waitall_on_empty_requests_is_noop():
    from paper_2107_00555_b200 import simrun

    out, _ = simrun.sim_run(_doc("dist_waitall_empty"), (2, 1),
                            _ctx({"N": 4}, {"A": np.zeros(4)}))
    assert out["A"][0] == 1.0


def test_rank_divergent_collectives_detected():
    """test_dist.py:309-326."""
    from paper_2107_00555_b200 import simrun

    with pytest.raises(simrun.CollectiveOrderError):
        simrun.sim_run(_doc("dist_divergent"), (2, 1),
                       _ctx({"N": 8}, {"A": np.arange(8.0), "B": np.arange(8.0),
                                       "C": np.zeros(8)}),
                       [{"me": 0}, {"me": 1}])


@pytest.mark.parametrize("P", [1, 2, 4])
def test_local_view_jacobi2d_equals_global(P):
    """test_dist.py:288-306: the explicit-halo local-view jacobi_2d on P
    ranks equals the shared-memory program bitwise (same op order)."""
    from oracle import interp_ref
    from paper_2107_00555_b200 import comm, sdfg, simrun

    N, T = 10, 4
    rng = np.random.default_rng(5)
    A, B = rng.uniform(-1, 1, (N, N)), rng.uniform(-1, 1, (N, N))
    ref = interp_ref.interpret(sdfg.from_dict(_doc("jacobi_2d")), {"N": N, "TSTEPS": T},
                               {"A": A.copy(), "B": B.copy()})
    binds, wins = [], []
    for r in range(P):
        b, w = comm.jacobi2d_rank_setup(N, P, r)
        binds.append(dict(b, TSTEPS=T))
        wins.append(w)
    lnx = binds[0]["lNx"]
    # every rank starts from its own window of the global arrays
    stores = [{"A": A[lo:hi].copy(), "B": B[lo:hi].copy()} for lo, hi in wins]
    sim = simrun.RankSim(_doc("jacobi2d_local"), (P, 1), _ctx({"lNx": lnx, "N": N}, {}),
                         binds, stores=stores)
    try:
        sim.run()
        for r in range(P):
            lo, hi = wins[r]
            m = sim.ranks[r].machine
            for k in ("A", "B"):
                got = m.store[k]
                assert np.array_equal(got[1:-1, :], ref[k][lo + 1:hi - 1, :]), (r, k)
    finally:
        sim.close()


@pytest.mark.parametrize("gdims", [(1, 1), (2, 1), (1, 2), (2, 2)])
@pytest.mark.parametrize("bs", [1, 2, 3, 4])
def test_block_cyclic_roundtrip_on_device(gdims, bs):
    """pkg/tests/test_dist.py:328-376 on the B200 rank simulator:
    block_gather(block_scatter(A)) == A for block-cyclic layouts (uneven
    block size 3 included); each block of a rank moves by its own copy."""
    from test_distribute import _cyclic_bindings, _cyclic_doc

    from paper_2107_00555_b200 import simrun

    extent = 4
    A = np.random.default_rng(bs).uniform(-1, 1, (extent, extent))
    out, _ = simrun.sim_run(_cyclic_doc(extent, gdims, bs), gdims,
                            _ctx({}, {"A": A, "B": np.zeros_like(A)}),
                            _cyclic_bindings(extent, gdims, bs))
    assert np.array_equal(out["B"], A)


@pytest.mark.parametrize("gdims", [(1, 1), (2, 1), (1, 2), (2, 2)])
def test_local_view_benchmark_on_device(gdims):
    """pkg/tests/test_dist.py:288-306 / test_acceptance.py:285-317 through
    dist.benchmark.run on the B200: equal to the shared-memory jacobi_2d
    (bitwise: same op order), 8 posted sends per rank per step on 2x2."""
    from oracle import interp_ref
    from paper_2107_00555_b200 import sdfg
    from paper_2107_00555_b200.dist import ProcessGrid, benchmark as BM

    n, tsteps = 8, 4
    rng = np.random.default_rng(13)
    A, B = rng.uniform(-1, 1, (n, n)), rng.uniform(-1, 1, (n, n))
    ref = interp_ref.interpret(sdfg.load(GOLDEN / "graphs" / "jacobi_2d.raw.json"),
                               {"N": n, "TSTEPS": tsteps}, {"A": A.copy(), "B": B.copy()})
    out, instr = BM.run(n, tsteps, ProcessGrid(gdims), A.copy(), B.copy())
    assert np.array_equal(out["A"], ref["A"]) and np.array_equal(out["B"], ref["B"])
    for c in instr["per_rank"].values():
        assert c["messages_posted"] == 8 * (tsteps - 1)
