"""Sliding-window contraction spot check: conv2d_bias through interpret() at
three shapes (generic path, BK = 12 and BK = 60 windows) against a numpy
einsum (dev tool)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2107_00555_b200 import ExecContext, interpret, sdfg
g = sdfg.load("tests/golden/graphs/conv2d_bias.raw.json")
for (NB, H, W, CI, CO, K) in ((1, 12, 300, 3, 16, 5), (2, 30, 40, 3, 16, 4), (8, 40, 256, 3, 16, 20)):
    HO, WO = H - K + 1, W - K + 1
    rng = np.random.default_rng(0)
    inp = rng.uniform(-1, 1, (NB, H, W, CI)); w = rng.uniform(-1, 1, (K, K, CI, CO)); b = rng.uniform(-1, 1, CO)
    out0 = np.zeros((NB, HO, WO, CO))
    syms = dict(NB=NB, H=H, W=W, CI=CI, CO=CO, K=K, HO=HO, WO=WO)
    r = interpret(g, ExecContext(bindings=syms).bind_inputs({"inp": inp, "w": w, "bias": b, "out": out0}))["out"]
    ref = np.broadcast_to(b, out0.shape).copy()
    for ki in range(K):
        for kj in range(K):
            ref += np.einsum("nijc,cd->nijd", inp[:, ki:ki + HO, kj:kj + WO, :], w[ki, kj])
    err = np.abs(r - ref) / np.maximum(np.abs(ref), 1)
    bad = np.argwhere(err > 1e-10)
    print(syms, err.max(), len(bad), bad[:5].tolist())
