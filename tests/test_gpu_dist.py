"""Multi-GPU plumbing checks that fit on ONE GPU: libb2's NCCL communicator
(world size 1, send/recv to self inside a captured CUDA graph) and the slab
runner's capture path.  The multi-rank logic itself is covered by the gloo
tests in test_dist.py."""

import ctypes
import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import torch
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
    _ = torch


def test_nccl_self_p2p_captured_in_graph(pg):
    from paper_2107_00555_b200 import dist, runtime as rt

    rt.device(0)
    L = rt.lib()
    comm = dist.NcclComm(0, 1)
    n = 1 << 16
    a = np.arange(n, dtype=np.float64)
    pa, pb = ctypes.c_void_p(), ctypes.c_void_p()
    rt.check(L.b2_malloc(ctypes.byref(pa), n * 8))
    rt.check(L.b2_malloc(ctypes.byref(pb), n * 8))
    s = ctypes.c_void_p()
    rt.check(L.b2_stream_create(ctypes.byref(s)))
    rt.check(L.b2_memcpy_h2d(pa, a.ctypes.data, n * 8, s))
    rt.check(L.b2_memset(pb, 0, n * 8, s))
    rt.check(L.b2_stream_sync(s))
    rt.check(L.b2_capture_begin(s))
    comm.p2p([(True, 0, pa.value, n * 8), (False, 0, pb.value, n * 8)], s.value)
    ge = ctypes.c_void_p()
    rt.check(L.b2_capture_end(s, ctypes.byref(ge)))
    rt.check(L.b2_graph_launch(ge, s))
    out = np.empty(n)
    rt.check(L.b2_memcpy_d2h(out.ctypes.data, pb, n * 8, s))
    rt.check(L.b2_stream_sync(s))
    assert np.array_equal(out, a)
    # a captured graph keeps NCCL work alive: destroy it before the communicator
    rt.check(L.b2_graph_destroy(ge))
    comm.close()


def test_slab_runner_single_rank_matches_oracle(pg):
    from oracle import kernels_np as K
    from paper_2107_00555_b200 import dist, sdfg

    g = sdfg.load(GOLDEN / "graphs" / "heat_3d.raw.json")
    syms = {"N": 40, "TSTEPS": 6}
    rng = np.random.default_rng(3)
    A = rng.uniform(-1, 1, (40, 40, 40))
    B = rng.uniform(-1, 1, (40, 40, 40))
    r = dist.SlabGpuRunner(g, syms, 0, 1, 0)
    r.load_inputs({"A": A, "B": B})
    r.run()
    out = r.gather({"A": A, "B": B})
    r.close()
    K.heat_3d_c(A, B, 6)
    assert np.array_equal(out["A"], A) and np.array_equal(out["B"], B)


@pytest.mark.parametrize("N", [40, 64])
def test_slab_runner_split_launch_bitwise(pg, N):
    """The overlapped launch path (boundary planes on a side stream, interior
    on the executor stream, joined inside the captured graph) forced on one
    rank: bitwise equal to the C oracle."""
    from oracle import kernels_np as K
    from paper_2107_00555_b200 import dist, sdfg

    g = sdfg.load(GOLDEN / "graphs" / "heat_3d.raw.json")
    syms = {"N": N, "TSTEPS": 5}
    rng = np.random.default_rng(N)
    A = rng.uniform(-1, 1, (N, N, N))
    B = rng.uniform(-1, 1, (N, N, N))
    r = dist.SlabGpuRunner(g, syms, 0, 1, 0, overlap=True, force_split=True)
    r.load_inputs({"A": A, "B": B})
    r.run()
    assert r.splits > 0
    out = r.gather({"A": A, "B": B})
    r.close()
    K.heat_3d_c(A, B, 5)
    assert np.array_equal(out["A"], A) and np.array_equal(out["B"], B)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_summa_single_rank_with_libb2_gemm(pg, dtype):
    """dist.Summa on a 1x1 grid with the libb2 GEMMs the SUMMA bench uses
    (DMMA f64 / tcgen05 3xTF32 f32), K cut into panels, C accumulated."""
    import torch

    from paper_2107_00555_b200 import dist, runtime as rt

    rt.device(0)
    L = rt.lib()
    n = 1024
    tdt = torch.float64 if dtype == "f64" else torch.float32
    fn = L.b2_gemm_f64 if dtype == "f64" else L.b2_gemm_f32
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.rand((n, n), dtype=tdt, device="cuda", generator=g) * 2 - 1
    b = torch.rand((n, n), dtype=tdt, device="cuda", generator=g) * 2 - 1
    c = torch.zeros((n, n), dtype=tdt, device="cuda")
    s = dist.Summa(dist.ProcessGrid((1, 1)), 0, n, n, n)

    def gemm(cc, pa, pb):
        stream = torch.cuda.current_stream().cuda_stream
        rt.check(fn(pa.shape[0], pb.shape[1], pa.shape[1], pa.data_ptr(), pa.stride(0), 1,
                    pb.data_ptr(), pb.stride(0), 1, cc.data_ptr(), cc.stride(0), 1,
                    rt.WCR_CODE["add"], stream))

    s.run(a, b, c, gemm, lambda shape: torch.empty(shape, dtype=tdt, device="cuda"))
    torch.cuda.synchronize()
    ref = a.double().cpu().numpy() @ b.double().cpu().numpy()
    got = c.double().cpu().numpy()
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= (1e-12 if dtype == "f64" else 1e-5), err


@pytest.mark.parametrize("dtype,n", [("f64", 1024), ("f32", 1024), ("f64", 768)])
def test_summa_device_data_plane_single_rank(pg, dtype, n):
    """dist.SummaDevice (libb2 data plane: split / pack once, NCCL panel
    broadcasts on a comm stream, panel GEMMs on the compute stream, one
    captured CUDA graph) on a 1x1 grid: C = A @ B, and a replay of the graph
    recomputes the same C."""
    import torch

    from paper_2107_00555_b200 import dist, runtime as rt

    rt.device(0)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(7)
    a = torch.rand((n, n), dtype=tdt, device="cuda", generator=g) * 2 - 1
    b = torch.rand((n, n), dtype=tdt, device="cuda", generator=g) * 2 - 1
    c = torch.full((n, n), 7.0, dtype=tdt, device="cuda")
    torch.cuda.synchronize()
    sd = dist.SummaDevice(dist.ProcessGrid((1, 1)), 0, n, n, n, dtype)
    try:
        sd.capture(a.data_ptr(), b.data_ptr(), c.data_ptr())
        sd.launch()
        rt.check(rt.lib().b2_stream_sync(sd.sc))
        first = c.clone()
        sd.launch()
        rt.check(rt.lib().b2_stream_sync(sd.sc))
        assert torch.equal(first, c)
        assert sd.kernels_per_call == (3 if dtype == "f32" else 2)
    finally:
        sd.close()
    ref = a.double().cpu().numpy() @ b.double().cpu().numpy()
    got = c.double().cpu().numpy()
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= (1e-12 if dtype == "f64" else 1e-5), err


def _peer_worker(rank, port, q):
    import ctypes

    import torch.distributed as tdist

    from paper_2107_00555_b200 import dist, runtime as rt, sdfg

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        rt.device(0)
        L = rt.lib()
        syms = {"N": 12, "TSTEPS": 2}
        g = sdfg.load(GOLDEN / "graphs" / "heat_3d.raw.json")
        plan = dist.slab_decompose(g, syms, 2)
        rng = np.random.default_rng(3)
        ptrs, rows, want = {}, {}, {}
        for c in sorted(plan.dist):
            full = rng.uniform(-1, 1, (12, 12, 12))
            lo, hi = plan.window[rank][c]
            buf = np.array(full[lo:hi], copy=True)
            for row_i in plan.owned[1 - rank][c] & set(range(lo, hi)):
                buf[row_i - lo] = np.nan  # only the peer's stores may fill these
            p = ctypes.c_void_p()
            rt.check(L.b2_malloc(ctypes.byref(p), buf.nbytes))
            rt.check(L.b2_memcpy_h2d(p, buf.ctypes.data, buf.nbytes, None))
            ptrs[c], rows[c], want[c] = p.value, 144, full[lo:hi]
        s = ctypes.c_void_p()
        rt.check(L.b2_stream_create(ctypes.byref(s)))

        def host_sync(peers, stream):
            rt.check(L.b2_stream_sync(stream))
            tdist.barrier()

        ph = dist.PeerHalo(plan, rank, ptrs, rows, sync=host_sync)
        ops = []
        for c in sorted(plan.dist):
            sends, recvs = plan.transfers(c, rank)
            ops += [(True, p_, c, lo, hi) for p_, lo, hi in sends]
            ops += [(False, p_, c, lo, hi) for p_, lo, hi in recvs]
        n = ph.exchange(ops, s.value)
        ok = n > 0
        for c in sorted(plan.dist):
            got = np.empty_like(want[c])
            rt.check(L.b2_memcpy_d2h(got.ctypes.data, ptrs[c], got.nbytes, None))
            ok = ok and np.array_equal(got, want[c])
        tdist.barrier()
        ph.close()
        tdist.barrier()
        for p in ptrs.values():
            L.b2_free(p)
        q.put((rank, bool(ok), n))
    finally:
        tdist.destroy_process_group()


def test_peer_halo_two_processes_one_gpu():
    """dist.PeerHalo's data path: two processes on the same GPU map each
    other's slab buffers through CUDA IPC and store the halo rows the other
    reads (host-side sync instead of the NCCL tokens, which need two GPUs);
    afterwards every window equals the global array."""
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
