"""The paper's §5 kernel comparison on the B200 (the reference's
harness bench.hpp:133-313 and `swdg bench`, tools/swdg_main.cpp:81-110).

For N = 1..15 at a fixed memory load (elements_for_budget, bench.hpp:296-301: 10
nodal fields per element; the paper filled the GTX 1080's 8 GB, the default here
is the same 8 GiB): the split-form and the standard volume kernels
(swdg_gpu_volume_kernel, csrc/kernels_bench.cu) timed with CUDA events, the
device-to-device copy bandwidth of the same byte count (bench.hpp:216-229), and
the table of bench.hpp:305-313 plus GFLOPS and the split/standard runtime ratio:

    N;K;DOFs;evals_split;evals_std;flops_split;flops_std;t_split;t_std;t_memcpy;bw_eff;roofline

Operation counts are the closed forms of bench::count_ops (bench.hpp:160-192):
evals_split = 2 (N+1)^3 K, evals_std = 2 (N+1)^2 K, F_ref = flops_split =
(88 (N+1) + 5) (N+1)^2 K, flops_std = (12 (N+1) + 38) (N+1)^2 K
(tests/test_paper_bench.py pins them to the reference's CountReal counter).
The roofline column is min(memcopy roofline, FP64 peak) -- the combined
roofline of bench.hpp:252-253 with the measured DFMA peak as the ceiling.

    python -m paper_1804_02221_b200.paper_bench [--budget-gb 8] [--reps 50] [--degrees 1-15]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os

from . import swdg


def counts(N: int, K: int):
    """bench::count_ops closed forms: evals_split, evals_std, flops_split, flops_std"""
    n1 = N + 1
    return (2 * n1 ** 3 * K, 2 * n1 ** 2 * K, (88 * n1 + 5) * n1 * n1 * K,
            (12 * n1 + 38) * n1 * n1 * K)


def elements_for_budget(N: int, budget_bytes: int) -> int:
    """bench.hpp:296-301"""
    return max(1, budget_bytes // (10 * (N + 1) ** 2 * 8))


def kernel_bytes_rw(N: int, K: int) -> int:
    """bench.hpp:196-202: 3 state + 4 metric fields read, 3 written, plus D"""
    np_ = (N + 1) ** 2
    return ((3 + 4) * np_ * K + np_ + 3 * np_ * K) * 8


def _fn():
    L = swdg.lib()
    f = L.swdg_gpu_volume_kernel
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_int, C.c_int64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                  C.c_double, C.c_void_p]
    return f


def buffers(N: int, K: int, seed: int = 20250810):
    """KernelBuffers::init (bench.hpp:108-131) on the device: a seeded rough wet
    field h ~ U(0.5, 2), hu, hv = h U(-1, 1), uniform-element metrics
    y_eta = x_xi = 0.5, x_eta = y_xi = 0; outputs zeroed.  (The reference seeds
    std::mt19937; torch's generator gives the same distribution.)"""
    import torch
    n = K * (N + 1) ** 2
    g = torch.Generator(device="cuda").manual_seed(seed)
    h = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 1.5 + 0.5
    hu = h * (torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
    hv = h * (torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
    ye = torch.full((n,), 0.5, dtype=torch.float64, device="cuda")
    xe = torch.zeros(n, dtype=torch.float64, device="cuda")
    yx = torch.zeros(n, dtype=torch.float64, device="cuda")
    xx = torch.full((n,), 0.5, dtype=torch.float64, device="cuda")
    outs = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    return [h, hu, hv, ye, xe, yx, xx], outs


def run_kernel(kind: int, N: int, K: int, ins, outs, g: float = 9.81, stream=None):
    f = _fn()
    pin = (C.c_void_p * 7)(*(t.data_ptr() for t in ins))
    pout = (C.c_void_p * 3)(*(t.data_ptr() for t in outs))
    rc = f(kind, N, K, pin, pout, g, C.c_void_p(stream))
    if rc != swdg.SWDG_OK:
        raise swdg.CudaError(f"swdg_gpu_volume_kernel rc={rc}")


def time_row(N: int, budget: int, reps: int, fp64_peak: float):
    import torch
    K = elements_for_budget(N, budget)
    ins, outs = buffers(N, K)
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def timed(fn):
        fn()  # warm-up
        torch.cuda.synchronize()
        ev[0].record(stream)
        for _ in range(reps):
            fn()
        ev[1].record(stream)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) * 1e-3 / reps

    t_split = timed(lambda: run_kernel(0, N, K, ins, outs, stream=stream.cuda_stream))
    t_std = timed(lambda: run_kernel(1, N, K, ins, outs, stream=stream.cuda_stream))
    bytes_rw = kernel_bytes_rw(N, K)
    # memcopy baseline (bench.hpp:216-229): a buffer of half the traffic copied
    src = torch.empty(bytes_rw // 2 // 8, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    t_mem = timed(lambda: dst.copy_(src))
    del src, dst, ins, outs
    torch.cuda.empty_cache()
    es, estd, fs, fstd = counts(N, K)
    bw_mem = bytes_rw / t_mem
    roof_mem = fs / bytes_rw * bw_mem
    roofline = min(roof_mem, fp64_peak * 1e12)
    return dict(N=N, K=K, DOFs=3 * K * (N + 1) ** 2, evals_split=es, evals_std=estd,
                flops_split=fs, flops_std=fstd, t_split=t_split, t_std=t_std, t_memcpy=t_mem,
                bw_eff=bytes_rw / t_split, roofline=roofline,
                gflops_split=fs / t_split / 1e9, gflops_std=fstd / t_std / 1e9,
                runtime_ratio=t_split / t_std, flop_ratio=fs / fstd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget-gb", type=float, default=8.0)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--degrees", default="1-15")
    ap.add_argument("--fp64-peak", type=float, default=36.8,
                    help="TFLOP/s ceiling (profiles/r01_fp64_peak.json, DFMA microbenchmark)")
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    lo, _, hi = a.degrees.partition("-")
    degrees = range(int(lo), int(hi or lo) + 1)
    budget = int(a.budget_gb * (1 << 30))
    rows = [time_row(N, budget, a.reps, a.fp64_peak) for N in degrees]
    print("N;K;DOFs;evals_split;evals_std;flops_split;flops_std;t_split;t_std;t_memcpy;bw_eff;"
          "roofline;gflops_split;gflops_std;t_split/t_std;flops_split/flops_std")
    for r in rows:
        print(f"{r['N']};{r['K']};{r['DOFs']};{r['evals_split']};{r['evals_std']};"
              f"{r['flops_split']};{r['flops_std']};{r['t_split']:.6e};{r['t_std']:.6e};"
              f"{r['t_memcpy']:.6e};{r['bw_eff']:.6e};{r['roofline']:.6e};"
              f"{r['gflops_split']:.1f};{r['gflops_std']:.1f};{r['runtime_ratio']:.3f};"
              f"{r['flop_ratio']:.3f}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump(dict(budget_bytes=budget, reps=a.reps, rows=rows), f, indent=1)


if __name__ == "__main__":
    main()
