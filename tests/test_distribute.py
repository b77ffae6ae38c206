"""Distribution passes (distribute.py) — the reference's missing
``sdfgkit.dist`` transformations, restated from SPEC.md:505-603 — checked on
CPU through the rank-simulator oracle (oracle/dist_ref.py) against the
shared-memory interpreter oracle, with the properties pkg/tests/test_dist.py
pins (soundness on the 11 distributed-corpus kernels x grids {1x1, 2x1,
2x2}, Fig. 7 shape, redundant gather-scatter removal, no removal when T is
read elsewhere or distributions differ, uneven extents rejected)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, rel_err

# desk-scale extents divisible by every tested rank count (test_dist.py:19-31)
DIST_SYMBOLS = {
    "atax": {"M": 8, "N": 4},
    "bicg": {"N": 8, "M": 4},
    "doitgen": {"NR": 4, "NQ": 4, "NP": 8},
    "gemm": {"NI": 4, "NJ": 8, "NK": 8},
    "gemver": {"N": 8},
    "gesummv": {"N": 8},
    "jacobi_1d": {"N": 10, "TSTEPS": 4},
    "jacobi_2d": {"N": 6, "TSTEPS": 4},
    "k2mm": {"NI": 4, "NJ": 8, "NK": 8, "NL": 4},
    "k3mm": {"NI": 4, "NJ": 8, "NK": 8, "NM": 4, "NL": 8},
    "mvt": {"N": 8},
}
GRIDS = [(1, 1), (2, 1), (2, 2)]


def _doc(name):
    return json.loads((GOLDEN / "graphs" / f"{name}.raw.json").read_text())


def _inputs(g, syms, seed=31):
    from paper_2107_00555_b200 import symexpr

    rng = np.random.default_rng(seed)
    out = {}
    for n, c in g.containers.items():
        if not c.transient:
            shp = tuple(symexpr.evaluate(d, syms) for d in c.shape)
            out[n] = rng.uniform(-1, 1, shp) if shp else np.float64(rng.uniform(0.5, 1.5))
    return out


def _shared(name, syms, ins):
    from oracle import interp_ref
    from paper_2107_00555_b200 import sdfg

    return interp_ref.interpret(sdfg.from_dict(_doc(name)), syms,
                                {k: np.array(v) for k, v in ins.items()})


@pytest.mark.parametrize("gdims", GRIDS)
@pytest.mark.parametrize("name", sorted(DIST_SYMBOLS))
def test_distribution_soundness(name, gdims):
    """test_dist.py:194-200: distributed == shared memory (<= 1e-12 here;
    the reference allows 1e-6)."""
    from oracle import dist_ref
    from paper_2107_00555_b200 import distribution as D, sdfg

    syms = DIST_SYMBOLS[name]
    ins = _inputs(sdfg.from_dict(_doc(name)), syms)
    doc, _ = D.distribution_pipeline(_doc(name), gdims)
    out, _ = dist_ref.sim_run(doc, gdims, syms, {k: np.array(v) for k, v in ins.items()})
    ref = _shared(name, syms, ins)
    assert max(rel_err(out[k], ref[k]) for k in ref) <= 1e-12


def test_distributed_graphs_validate():
    from paper_2107_00555_b200 import distribution as D, sdfg, validate

    for name in DIST_SYMBOLS:
        for gd in GRIDS:
            doc, _ = D.distribution_pipeline(_doc(name), gd)
            assert validate.errors(sdfg.from_dict(doc)) == [], (name, gd)


def test_fig7_shape():
    """tmp0 = alpha*A on 2x2 -> Bcast(alpha), BlockScatter(A),
    local map, BlockGather(tmp0)."""
    from paper_2107_00555_b200 import distribution as D

    doc, rep = D.distribute(_doc("dist_alpha"), (2, 2))
    kinds = sorted(n["kind"] for st in doc["states"] for n in st["nodes"]
                   if n["type"] == "library")
    assert kinds == ["bcast", "block_gather", "block_scatter"]
    assert rep["distribute_elementwise"] == 1
    locs = [c for c in doc["containers"] if c.get("storage") == "distributed_local"]
    assert len(locs) == 3  # alpha, A block, T block


def test_flat_scatter_chunks():
    """test_dist.py:43-52: a dense 1-D map scatters flat chunks."""
    from oracle import dist_ref
    from paper_2107_00555_b200 import distribution as D

    doc, _ = D.distribution_pipeline(_doc("dist_flat"), (4, 1))
    kinds = {n["kind"] for st in doc["states"] for n in st["nodes"] if n["type"] == "library"}
    assert kinds == {"scatter", "gather"}
    A = np.arange(8.0)
    out, cnt = dist_ref.sim_run(doc, (4, 1), {"N": 8}, {"A": A, "B": np.zeros(8)})
    assert np.array_equal(out["B"], A)


def test_uneven_block_extent_fails():
    """test_dist.py:64-73: no implicit padding."""
    from paper_2107_00555_b200 import distribution as D

    doc, _ = D.distribution_pipeline(_doc("dist_flat"), (4, 1))
    with pytest.raises(D.DistError, match="divisible|covered"):
        D.local_bindings(doc, (4, 1), {"N": 6}, 0)


def _colls(doc):
    return sum(1 for st in doc["states"] for n in st["nodes"] if n["type"] == "library"
               and n["kind"] in ("scatter", "gather", "bcast", "block_scatter", "block_gather"))


def test_gemm_redundant_pairs_removed():
    """SPEC.md:563 / test_dist.py:216-262: every removed gather-scatter pair
    takes two collective nodes and two collective calls away, outputs
    bitwise unchanged.  (The reference pins 2 pairs on gemm: its first,
    flat-scattered statement never matches the 2-D product; here every
    2-D statement is block-distributed, so tmp0 / tmp1 / tmp2 all match.)"""
    from oracle import dist_ref
    from paper_2107_00555_b200 import distribution as D, sdfg

    syms = DIST_SYMBOLS["gemm"]
    full, _ = D.distribute(_doc("gemm"), (2, 2))
    red, _ = D.distribute(_doc("gemm"), (2, 2))
    rep = D.remove_redundant_comm(red)
    pairs = rep.get("remove_redundant_comm", 0)
    assert pairs == 3
    assert _colls(full) - _colls(red) == 2 * pairs
    ins = _inputs(sdfg.from_dict(_doc("gemm")), syms)
    o1, c1 = dist_ref.sim_run(full, (2, 2), syms, {k: np.array(v) for k, v in ins.items()})
    o2, c2 = dist_ref.sim_run(red, (2, 2), syms, {k: np.array(v) for k, v in ins.items()})
    assert c1[0]["collective_calls"] - c2[0]["collective_calls"] == 2 * pairs
    for k in o1:
        assert np.array_equal(o1[k], o2[k])


def test_global_read_elsewhere_not_removed():
    """test_dist.py:264-282: T read by two statements -> nothing removed."""
    from paper_2107_00555_b200 import distribution as D

    doc, _ = D.distribute(_doc("dist_two_readers"), (2, 1))
    assert D.remove_redundant_comm(doc).get("remove_redundant_comm", 0) == 0


def test_mismatched_distribution_not_removed():
    """T gathered flat (dense 1-D map) but re-scattered as a shifted view
    T[:-2]: different collectives / subsets -> kept; the
    frontend's dense temporary tmp0 (T[:-2] * 2.0, then copied into B[1:-1])
    is gathered and re-scattered flat with the same layout -> removed."""
    from oracle import dist_ref
    from paper_2107_00555_b200 import distribution as D, sdfg

    doc, rep = D.distribution_pipeline(_doc("dist_shifted"), (2, 1))
    assert rep.get("remove_redundant_comm", 0) == 1
    touching_T = [n["kind"] for st in doc["states"] for n in st["nodes"]
                  if n["type"] == "library"
                  and any(e.get("memlet", "").startswith("T[") for e in st["edges"]
                          if n["id"] in (e["src"], e["dst"]))]
    assert sorted(touching_T) == ["block_scatter", "gather"]
    syms = {"N": 10}
    ins = _inputs(sdfg.from_dict(_doc("dist_shifted")), syms)
    out, _ = dist_ref.sim_run(doc, (2, 1), syms, {k: np.array(v) for k, v in ins.items()})
    ref = _shared("dist_shifted", syms, ins)
    assert all(np.array_equal(out[k], ref[k]) for k in ref)


def test_single_rank_moves_no_bytes():
    """P = 1 -> every collective is a local copy."""
    from oracle import dist_ref
    from paper_2107_00555_b200 import distribution as D, sdfg

    syms = DIST_SYMBOLS["gemm"]
    doc, _ = D.distribution_pipeline(_doc("gemm"), (1, 1))
    ins = _inputs(sdfg.from_dict(_doc("gemm")), syms)
    _, cnt = dist_ref.sim_run(doc, (1, 1), syms, ins)
    assert cnt[0]["comm_bytes"] == 0 and cnt[0]["messages_posted"] == 0


def _cyclic_doc(extent, dims, bs):
    """A -> BLOCK_SCATTER -> L (lr x lc, distributed local) -> BLOCK_GATHER -> B
    with a block-cyclic distribution (pkg/tests/test_dist.py:328-376)."""
    attr = {"dist": {"grid": list(dims), "block": [str(bs), str(bs)], "scheme": "block_cyclic"}}
    full = f"[0:{extent - 1}:1, 0:{extent - 1}:1]"
    lfull = "[0:(lr - 1):1, 0:(lc - 1):1]"
    c = lambda n, shape, tr, st: {"name": n, "dtype": "f64", "shape": shape, "kind": "array",  # noqa: E731
                                  "transient": tr, "lifetime": "scope", "storage": st}
    return {"version": 1, "name": "cyc",
            "symbols": [{"name": "lr", "min": 0}, {"name": "lc", "min": 0}],
            "containers": [c("A", [str(extent)] * 2, False, "heap"),
                           c("B", [str(extent)] * 2, False, "heap"),
                           c("L", ["lr", "lc"], True, "distributed_local")],
            "states": [{"label": "s0", "nodes": [
                {"id": 0, "type": "access", "container": "A"},
                {"id": 1, "type": "library", "kind": "block_scatter", "name": "scatter", "attrs": attr},
                {"id": 2, "type": "access", "container": "L"},
                {"id": 3, "type": "library", "kind": "block_gather", "name": "gather", "attrs": attr},
                {"id": 4, "type": "access", "container": "B"}],
                "edges": [{"src": 0, "dst": 1, "dst_conn": "a", "memlet": "A" + full},
                          {"src": 1, "dst": 2, "src_conn": "out", "memlet": "L" + lfull},
                          {"src": 2, "dst": 3, "dst_conn": "a", "memlet": "L" + lfull},
                          {"src": 3, "dst": 4, "src_conn": "out", "memlet": "B" + full}]}],
            "transitions": [], "start": "s0"}


def _cyclic_bindings(extent, dims, bs):
    from paper_2107_00555_b200.dist import ProcessGrid, block_indices

    grid = ProcessGrid(dims)
    out = []
    for r in range(grid.size):
        co = grid.coords(r)
        i, j = co[0], (co[1] if len(co) == 2 else 0)
        out.append({"lr": len(block_indices(extent, dims[0], i, bs)),
                    "lc": len(block_indices(extent, dims[1], j, bs))})
    return out


@pytest.mark.parametrize("gdims", [(1, 1), (2, 1), (2, 2)])
@pytest.mark.parametrize("scheme_block", [1, 2, None])
def test_block_indices_cover_every_cell_once(gdims, scheme_block):
    """pkg/tests/test_dist.py:66-85: ownership covers every cell exactly once."""
    from paper_2107_00555_b200.dist import ProcessGrid, block_indices

    grid, extent = ProcessGrid(gdims), 4
    blocks = [scheme_block or -(-extent // d) for d in gdims]
    owned = np.zeros((extent, extent), dtype=int)
    for r in range(grid.size):
        i, j = grid.coords(r)
        for x in block_indices(extent, gdims[0], i, blocks[0]):
            for y in block_indices(extent, gdims[1], j, blocks[1]):
                owned[x, y] += 1
    assert np.all(owned == 1)


@pytest.mark.parametrize("gdims", [(1, 1), (2, 1), (1, 2), (2, 2)])
@pytest.mark.parametrize("bs", [1, 2, 3, 4])
def test_block_cyclic_roundtrip_oracle(gdims, bs):
    """pkg/tests/test_dist.py:328-376: block_gather(block_scatter(A)) == A for
    block-cyclic layouts (block sizes 1, 2, 3 — uneven — and the extent) in
    the CPU rank-simulator oracle."""
    from oracle import dist_ref

    extent = 4
    A = np.random.default_rng(bs).uniform(-1, 1, (extent, extent))
    out, _ = dist_ref.sim_run(_cyclic_doc(extent, gdims, bs), gdims, {},
                              {"A": A, "B": np.zeros_like(A)},
                              rank_bindings=_cyclic_bindings(extent, gdims, bs))
    assert np.array_equal(out["B"], A)


def test_benchmark_program_text_is_the_compiled_one():
    from conftest import GOLDEN as _G  # noqa: F401
    import pathlib

    from paper_2107_00555_b200.dist import benchmark as BM

    root = pathlib.Path(__file__).resolve().parent.parent
    assert BM.JACOBI2D_LOCAL_VIEW == (root / "programs" / "jacobi2d_local_view.dpy").read_text()
    pkg = json.loads((root / "paper_2107_00555_b200" / "dist" / "jacobi2d_local_view.json").read_text())
    gold = json.loads((GOLDEN / "graphs" / "jacobi2d_local_view.raw.json").read_text())
    assert pkg == gold


@pytest.mark.parametrize("gdims", [(1, 1), (2, 1), (1, 2), (2, 2)])
def test_local_view_benchmark_oracle(gdims):
    """pkg/tests/test_dist.py:288-306 on the CPU rank-simulator oracle: the
    local-view jacobi_2d (dist.benchmark) equals the shared-memory program
    bitwise, and a 2x2 grid posts exactly 8 sends per rank per step (four
    directions, PROC_NULL on the global boundary)."""
    from oracle import dist_ref, interp_ref
    from paper_2107_00555_b200.dist import benchmark as BM

    n, tsteps = 8, 4
    rng = np.random.default_rng(5)
    A, B = rng.uniform(-1, 1, (n, n)), rng.uniform(-1, 1, (n, n))
    ref = interp_ref.interpret(sdfg_load("jacobi_2d"), {"N": n, "TSTEPS": tsteps},
                               {"A": A.copy(), "B": B.copy()})
    wins = BM.windows(n, gdims)
    stores = [{"A": A[w].copy(), "B": B[w].copy()} for w in wins]
    outs, cnt = dist_ref.sim_run(BM.build_graph(), gdims, {"TSTEPS": tsteps}, {},
                                 rank_bindings=BM.rank_bindings(n, gdims, tsteps),
                                 rank_stores=stores, all_outputs=True)
    gotA, gotB = A.copy(), B.copy()
    for r, (rs, cs) in enumerate(wins):
        inner = (slice(rs.start + 1, rs.stop - 1), slice(cs.start + 1, cs.stop - 1))
        gotA[inner] = outs[r]["A"][1:-1, 1:-1]
        gotB[inner] = outs[r]["B"][1:-1, 1:-1]
    assert np.array_equal(gotA, ref["A"]) and np.array_equal(gotB, ref["B"])
    for c in cnt.values():
        assert c["messages_posted"] == 8 * (tsteps - 1)


def sdfg_load(name):
    from paper_2107_00555_b200 import sdfg

    return sdfg.load(GOLDEN / "graphs" / f"{name}.raw.json")


def test_reference_dist_import_surface():
    """Every name pkg/tests/test_dist.py:5-10 imports from sdfgkit.dist,
    .dist.benchmark and .dist.layout exists under paper_2107_00555_b200.dist."""
    from paper_2107_00555_b200.dist import (  # noqa: F401
        DeadlockError, Distribution, ProcessGrid, RankSim, distribute,
        distribution_pipeline, remove_redundant_comm, sim_run,
    )
    from paper_2107_00555_b200.dist.benchmark import (  # noqa: F401
        JACOBI2D_LOCAL_VIEW, build_graph, rank_bindings, run,
    )
    from paper_2107_00555_b200.dist.layout import (  # noqa: F401
        SCHEME_BLOCK, SCHEME_BLOCK_CYCLIC, block_indices,
    )
    d = Distribution(ProcessGrid((2, 2)), [2, 2], SCHEME_BLOCK_CYCLIC)
    assert d.attr() == {"grid": [2, 2], "block": ["2", "2"], "scheme": "block_cyclic"}


def _ref_serializer():
    import importlib
    import pathlib
    import sys

    root = pathlib.Path(__file__).resolve().parent.parent
    for p in (root / "baseline" / "_ref", pathlib.Path("/root/reference/pkg/src")):
        if (p / "sdfgkit").exists() and str(p) not in sys.path:
            sys.path.insert(0, str(p))
    try:
        return importlib.import_module("sdfgkit.serialize")
    except ImportError:
        pytest.skip("reference package not installed (baseline/_ref)")


@pytest.mark.parametrize("gdims", [(2, 1), (2, 2)])
def test_passes_rewrite_a_reference_sdfg_in_place(gdims):
    """The reference's calling convention (test_dist.py:36-52, 216-262): the
    passes mutate the reference Sdfg they are given and return a report with
    .applications; the rewritten object validates in the reference and runs
    distributed (rank-simulator oracle) to the shared-memory result."""
    from oracle import dist_ref
    from paper_2107_00555_b200 import distribution as D, sdfg

    ser = _ref_serializer()
    doc = _doc("gemm")
    g = ser.from_dict(doc)
    rep = D.distribution_pipeline(g, gdims)
    assert rep.applications.get("expand_matmul_distributed", 0) == 1
    assert not [d for d in g.validate() if d.severity == "error"]
    syms = DIST_SYMBOLS["gemm"]
    ins = _inputs(sdfg.from_dict(doc), syms)
    out, _ = dist_ref.sim_run(g, gdims, syms, {k: np.array(v) for k, v in ins.items()})
    ref = _shared("gemm", syms, ins)
    assert max(rel_err(out[k], ref[k]) for k in ref) <= 1e-12
