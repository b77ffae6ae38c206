"""Compile extra programs with the REFERENCE frontend (and passes) into
schema-v1 graphs (run here, where /root/reference exists):

    python tests/golden/make_extra_graphs.py

Local-view (explicit message passing) programs:

programs/halo_pair.dpy      column exchange between two ranks (the pattern of
                            pkg/tests/test_dist.py:105-140)
programs/jacobi2d_local.dpy jacobi_2d with rows block-distributed and explicit
                            halo exchange (the SPEC.md:580 local-view example)
programs/overlap_recv.dpy   two outstanding receives into the same elements
                            (race diagnostic)
programs/block_roundtrip.dpy block_scatter -> local map -> block_gather
                            (SPEC.md:532-534 round trip)
"""

import json
import os
import pathlib
import sys

REF = pathlib.Path(os.environ.get("REF_PKG", "/root/reference/pkg"))
HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REF / "src"))

from sdfgkit import frontend  # noqa: E402
from sdfgkit.serialize import to_dict  # noqa: E402

for name in ("halo_pair", "jacobi2d_local", "overlap_recv", "block_roundtrip",
             "jacobi2d_local_view"):
    g, diags = frontend.compile_source((REPO / "programs" / f"{name}.dpy").read_text())
    errs = [d for d in diags if d.severity == "error"]
    assert not errs, errs
    out = HERE / "graphs" / f"{name}.raw.json"
    out.write_text(json.dumps(to_dict(g), indent=1) + "\n")
    print("wrote", out)
    if name == "jacobi2d_local_view":  # dist.benchmark's program graph (package data)
        pkg = REPO / "paper_2107_00555_b200" / "dist" / "jacobi2d_local_view.json"
        pkg.write_text(json.dumps(to_dict(g), indent=1) + "\n")
        print("wrote", pkg)

# Interpreter-contract programs (the cases of pkg/tests/test_interp.py:52-121,
# written here; compiled by the reference frontend, tile_wcr by its autoopt)
from sdfgkit import autoopt  # noqa: E402

CONTRACT = {
    "oob_read": "def f(A: f64[N], B: f64[N], K: i64):\n    B[0] = A[K]\n",
    "tiled_red": "def red(s: f64, A: f64[N]):\n    for i in map[0:N]:\n        s += A[i]\n",
    "bicg_head": "def bicg(A: f64[N, M], s: f64[M], q: f64[N], p: f64[M], r: f64[N]):\n"
                 "    s[:] = r @ A\n",
    "bicg_tail": "def bicg(A: f64[N, M], s: f64[M], q: f64[N], p: f64[M], r: f64[N]):\n"
                 "    q[:] = A @ p\n",
    # a loop whose branch condition reads a scalar container updated inside
    # the loop (interp.py:265-274: conditions may read 0-d containers)
    "branchy": "def branchy(TSTEPS: i32, x: f64[N], s: f64):\n"
               "    for t in range(TSTEPS):\n"
               "        if s > 0.0:\n"
               "            x[:] = x * 0.5\n"
               "            s = s - 1.0\n"
               "        else:\n"
               "            x[:] = x + 1.0\n",
}
for name, src in CONTRACT.items():
    g, diags = frontend.compile_source(src)
    assert g is not None, diags
    if name == "tiled_red":
        autoopt.tile_wcr(g, 16)
    out = HERE / "graphs" / f"{name}.raw.json"
    out.write_text(json.dumps(to_dict(g), indent=1) + "\n")
    print("wrote", out)

# Distribution-pipeline / rank-simulator programs (the cases of
# pkg/tests/test_dist.py:41-95, 143-180, 264-282, 348-366, written here)
DIST = {
    "dist_flat": "def f(A: f64[N], B: f64[N]):\n    B[:] = A + 0.0\n",
    "dist_alpha": "def f(alpha: f64, A: f64[N, M], T: f64[N, M]):\n    T[:] = alpha * A\n",
    "dist_two_readers": ("def f(A: f64[N], B: f64[N], C: f64[N]):\n"
                         "    T = zeros(N)\n"
                         "    T[:] = A + 1.0\n"
                         "    B[:] = T * 2.0\n"
                         "    C[:] = T + 3.0\n"),
    "dist_shifted": ("def f(A: f64[N], B: f64[N]):\n"
                     "    T = zeros(N)\n"
                     "    T[:] = A + 1.0\n"
                     "    B[1:-1] = T[:-2] * 2.0\n"),
    "dist_unmatched_send": ("def f(A: f64[lNx + 2, lNy + 2], peer: i32):\n"
                            "    req = requests(1)\n"
                            "    comm_isend(A[1:-1, 1], peer, 3, req[0])\n"
                            "    comm_waitall(req)\n"),
    "dist_missing_send": ("def f(A: f64[lNx + 2, lNy + 2], peer: i32):\n"
                          "    req = requests(1)\n"
                          "    comm_irecv(A[1:-1, 0], peer, 3, req[0])\n"
                          "    comm_waitall(req)\n"),
    "dist_waitall_empty": ("def f(A: f64[N]):\n"
                           "    req = requests(4)\n"
                           "    comm_waitall(req)\n"
                           "    A[0] = 1.0\n"),
    "dist_divergent": ("def f(A: f64[N], B: f64[N], C: f64[N], me: i32):\n"
                       "    la = zeros(N // 2)\n"
                       "    if me < 1:\n"
                       "        la[:] = block_scatter(A)\n"
                       "    else:\n"
                       "        la[:] = block_scatter(B)\n"
                       "    C[0:N // 2] = block_gather(la)\n"),
}
for name, src in DIST.items():
    g, diags = frontend.compile_source(src)
    errs = [d for d in diags if d.severity == "error"]
    assert g is not None and not errs, (name, [str(d) for d in diags])
    out = HERE / "graphs" / f"{name}.raw.json"
    out.write_text(json.dumps(to_dict(g), indent=1) + "\n")
    print("wrote", out)
