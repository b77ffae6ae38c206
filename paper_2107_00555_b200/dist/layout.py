"""Block and block-cyclic layouts of the distribution collectives
(BlockScatter / BlockGather; the reference's
``sdfgkit.dist.layout`` API used by pkg/tests/test_dist.py:66-85, 328-376).

A distribution splits array dim d over grid dim d (a 1-D grid splits the
first dim; trailing unit grid dims are dropped for lower-rank arrays).
``block``: one contiguous block per rank, the extent must be divisible (no
implicit padding).  ``block_cyclic``: blocks of size b dealt round-robin;
uneven extents are allowed.  A rank's local array is the
concatenation of its blocks along every dim."""

from __future__ import annotations

SCHEME_BLOCK = "block"
SCHEME_BLOCK_CYCLIC = "block_cyclic"


class LayoutError(RuntimeError):
    pass


def block_indices(extent: int, griddim: int, coord: int, block: int | None = None) -> list:
    """Indices of ``extent`` owned by ``coord`` of ``griddim``: contiguous
    near-equal blocks (block=None) or block-cyclic with block size ``block``."""
    if block is None:
        lo = extent * coord // griddim
        hi = extent * (coord + 1) // griddim
        return list(range(lo, hi))
    idx = []
    for start in range(coord * block, extent, griddim * block):
        idx.extend(range(start, min(start + block, extent)))
    return idx


def dim_runs(extent: int, griddim: int, coord: int, scheme: str = SCHEME_BLOCK,
             block: int | None = None) -> list:
    """[(global start, length, local start)] of the contiguous runs of one
    array dim owned by ``coord``."""
    if scheme == SCHEME_BLOCK:
        if extent % griddim:
            raise LayoutError(f"extent {extent} is not covered by grid dim {griddim} "
                              "(divisible block sizes required)")
        b = extent // griddim
        return [(coord * b, b, 0)]
    if scheme != SCHEME_BLOCK_CYCLIC:
        raise LayoutError(f"unknown distribution scheme {scheme!r}")
    b = int(block) if block else -(-extent // griddim)
    if b < 1:
        raise LayoutError(f"block size {b} < 1")
    out, loc = [], 0
    for start in range(coord * b, extent, griddim * b):
        n = min(b, extent - start)
        out.append((start, n, loc))
        loc += n
    return out


def block_runs(shape, grid_dims, coords, scheme: str = SCHEME_BLOCK, blocks=None) -> list:
    """Per array dim, the runs (``dim_runs``) of the rank at ``coords``."""
    grid_dims = list(grid_dims)
    while len(grid_dims) > len(shape) and grid_dims[-1] == 1:  # (P, 1) over a vector
        grid_dims.pop()
    if len(grid_dims) > len(shape):
        raise LayoutError(f"grid {tuple(grid_dims)} has more dims than the array {tuple(shape)}")
    out = []
    for d, n in enumerate(shape):
        if d < len(grid_dims):
            b = blocks[d] if blocks is not None and d < len(blocks) else None
            out.append(dim_runs(n, grid_dims[d], coords[d], scheme, b))
        else:
            out.append([(0, n, 0)])
    return out


def local_shape(runs) -> list:
    return [sum(n for _, n, _ in r) for r in runs]


class Distribution:
    """A container's distribution: grid, per-dimension
    block sizes (None = ceil(extent / grid dim)) and scheme.  ``attr()`` is
    the {"dist": ...} attribute of the BlockScatter / BlockGather nodes."""

    def __init__(self, grid, blocks=None, scheme: str = SCHEME_BLOCK):
        dims = getattr(grid, "dims", grid)
        self.grid = tuple(int(d) for d in dims)
        self.blocks = None if blocks is None else [str(b) for b in blocks]
        if scheme not in (SCHEME_BLOCK, SCHEME_BLOCK_CYCLIC):
            raise LayoutError(f"unknown distribution scheme {scheme!r}")
        self.scheme = scheme

    def attr(self) -> dict:
        return {"grid": list(self.grid), "block": self.blocks, "scheme": self.scheme}

    def __eq__(self, other):
        return isinstance(other, Distribution) and self.attr() == other.attr()

    def __repr__(self):
        return f"Distribution({self.grid}, {self.blocks}, {self.scheme!r})"
