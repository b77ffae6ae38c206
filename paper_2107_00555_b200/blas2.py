"""Pattern rules that fold MATMUL library nodes of BLAS-2 shape (and the
elementwise map that feeds one) into single rowpass-family passes.
Filled in by the rowpass family; the identity rule keeps the op list."""

from __future__ import annotations


def fuse(planner, ops):
    return ops
