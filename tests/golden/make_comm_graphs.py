"""Compile this repo's local-view (explicit message passing) programs with the
REFERENCE frontend into schema-v1 graphs (run here, where /root/reference
exists):

    python tests/golden/make_comm_graphs.py

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

for name in ("halo_pair", "jacobi2d_local", "overlap_recv", "block_roundtrip"):
    g, diags = frontend.compile_source((REPO / "programs" / f"{name}.dpy").read_text())
    errs = [d for d in diags if d.severity == "error"]
    assert not errs, errs
    out = HERE / "graphs" / f"{name}.raw.json"
    out.write_text(json.dumps(to_dict(g), indent=1) + "\n")
    print("wrote", out)
