"""Measured compute / on-chip ceilings for the roofline denominators that
MEASURED_PEAKS.json (HBM copy, bf16 GEMM) does not carry: DMMA f64, FP64 /
FP32 FMA, L2 read bandwidth (scripts/peaks/peaks.cu), plus library GEMM
ceilings through torch (cuBLAS DGEMM 16384^3 f64, cuBLAS TF32 8192^3).

    python scripts/peaks/measure_peaks.py [out.json]
"""

from __future__ import annotations

import json
import pathlib
import subprocess
import sys
import time

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))


def main():
    out = pathlib.Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / \
        "measured_peaks_extra.json"
    exe = HERE / "peaks"
    if not exe.exists() or exe.stat().st_mtime < (HERE / "peaks.cu").stat().st_mtime:
        subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o",
                        str(exe), str(HERE / "peaks.cu")], check=True)
    from bench import ClockSampler

    with ClockSampler() as clk:
        res = json.loads(subprocess.run([str(exe)], check=True, capture_output=True,
                                        text=True).stdout)
    res["clocks_microbench"] = clk.summary()
    import torch

    def gemm(n, dtype, tf32, reps):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        a = torch.rand(n, n, dtype=dtype, device="cuda") * 2 - 1
        b = torch.rand(n, n, dtype=dtype, device="cuda") * 2 - 1
        torch.matmul(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(reps):
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2 * n ** 3 / (best * 1e-3) / 1e12

    with ClockSampler() as clk:
        res["cublas_dgemm_16384_tflops"] = gemm(16384, torch.float64, False, 3)
    res["clocks_dgemm"] = clk.summary()
    with ClockSampler() as clk:
        res["cublas_tf32_8192_tflops"] = gemm(8192, torch.float32, True, 10)
    res["clocks_tf32"] = clk.summary()
    res["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    res["how"] = ("peaks.cu: best of 5 launches, CUDA events (dmma: mma.sync m16n8k4 f64, 8 "
                  "independent accumulators/warp, 4 CTAs x 256 thr per SM; fma: 8 chains/thread; "
                  "l2: 48 MB x 20 passes of 16-B __ldcg loads; hbm: 4 GB once); cuBLAS via "
                  "torch.matmul, best of N")
    out.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
