"""Multi-GPU execution (placeholder until the slab executor lands)."""


def bench_slab(args, W):
    raise NotImplementedError("multi-GPU slab execution is not implemented yet")
