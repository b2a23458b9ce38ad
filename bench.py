#!/usr/bin/env python
"""bench.py — TLR Cholesky time-to-solution on B200 (BASELINE.json config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tlrg|reference]
                    [--config cfg2] [--no-cpu-baseline]

A step is one full TLR Cholesky factorization (tlr_cholesky, factor.cpp:290-293)
of the 2D exponential covariance matrix N = 131,072, tile m = 512, eps = 1e-2,
bs = 16, root seed 12345, built on the device from the same
synthetic grid points the reference uses.  Inputs (1.17 GB) exceed L2, so no
flush is needed between steps.

value  : time-to-solution (s) per factorization, CUDA-event timed on the
         library stream, max over ranks, inputs resident in HBM.
e2e    : the same through the C ABI with host buffers: upload A, factorize,
         download L, per step.
Multi-GPU (torchrun, one process per GPU): every column's rank-sorted active
tiles are dealt round-robin over the ranks and the new panels are replicated
by an NCCL all-gather; the factor is bitwise identical to the
1-GPU one.  value = time of the whole factorization (max over ranks): strong
scaling of one fixed problem.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("TLR Cholesky FP64 time-to-solution (s) & TFLOP/s, 2D covariance N=131K "
          "ε=1e-2")

CONFIGS = {
    # name: (point kind, N, tile, eps, bs, kernel, ell, nugget, mode)
    "cfg1": (0, 16384, 256, 1e-6, 16, 0, 0.1, 0.0, 0),
    "cfg2": (0, 131072, 512, 1e-2, 16, 0, 0.1, 0.0, 0),
    "cfg3": (1, 65536, 512, 1e-4, 32, 1, 0.2, 1e-4, 1),
    "cfg4": (1, 262144, 1024, 1e-3, 32, 0, 0.2, 0.0, 0),
}
SEED = 12345
CPU_SAMPLE = "cfg2 family at N=32,768 (nb=64, m=512, eps=1e-2): full reference tlr_cholesky"


def workload_name(cfg):
    kind, n, b, eps, bs, kern, ell, nug, mode = CONFIGS[cfg]
    d = "2D" if kind == 0 else "3D"
    k = "exponential" if kern == 0 else "Gaussian"
    m = "Cholesky" if mode == 0 else "LDL^T"
    return f"{d} {k} covariance N={n} m={b} eps={eps:g} bs={bs} TLR {m} ({cfg})"


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.out = ""

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (getattr(self, "out", "") or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(path=os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                  "r01h_fused_ncu.txt")):
    """DRAM bytes of one fused-kernel launch from the committed ncu capture."""
    try:
        tot = 0
        for line in open(path):
            if line.startswith(("dram__bytes_read.sum:", "dram__bytes_write.sum:")):
                tot += int(float(line.split(":")[1].split()[0]))
        return tot or None
    except OSError:
        return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def dist_init(ws, backend):
    if ws <= 1:
        return None
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group(backend)
    return dist


def allmax(dist, x):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def measure_fp64_peak():
    """cuBLAS DGEMM 8192^3 via torch (burst, best of 5) — the FP64 roofline
    denominator (MEASURED_PEAKS.json has none for FP64)."""
    try:
        import torch
        a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
        b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
        for _ in range(2):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch.matmul(a, b)
            e.record()
            e.synchronize()
            best = max(best, 2 * 8192 ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12)
        del a, b
        torch.cuda.empty_cache()
        return best
    except Exception:
        return None


def problem_points(cfg):
    from paper_2108_11932_b200 import geometry as G
    kind, n, b = CONFIGS[cfg][:3]
    return G.kd_order(G.generate_points(kind, n, 0), b).matrix_order()


def cpu_baseline_sample():
    """Reference tlr_cholesky (oracle/_ref, unmodified sources) on a bounded
    sample of the workload family, all host threads."""
    from oracle import ref
    from paper_2108_11932_b200 import geometry as G
    ref.lib()
    n, b = 32768, 512
    pts = G.kd_order(G.generate_points(0, n, 0), b).matrix_order()
    A = ref.build(pts, 0, 0.1, 0.0, b, 1e-2, 0, 16, SEED)
    t = time.perf_counter()
    F = ref.factor(A, 0, bs=16, eps=1e-2, seed=SEED)
    dt = time.perf_counter() - t
    return dt, ref.lib().ref_max_threads(), F.stats().wall


def run_tlrg(args):
    ws, rank, local = dist_env()
    dist = dist_init(ws, "nccl")
    import numpy as np

    import paper_2108_11932_b200 as tg
    from paper_2108_11932_b200.tlr import build_tlr
    kind, n, b, eps, bs, kern, ell, nug, mode = CONFIGS[args.config]
    ctx = tg.Context(local)
    if dist is not None:
        # intra-column tile split over the ranks: NCCL id from
        # rank 0 over the torch process group, one communicator per GPU
        obj = [tg.nccl_unique_id(ctx) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.attach_nccl(rank, ws, obj[0])
    cfg = tg.AraConfig(block_samples=bs, eps=eps, seed=SEED)
    pts = problem_points(args.config)
    t0 = time.perf_counter()
    A0 = build_tlr(pts, kern, ell, nug, b, eps, compressor=0,
                   cfg=tg.AraConfig(block_samples=bs, seed=SEED), ctx=ctx)
    t_build = time.perf_counter() - t0
    mem = A0.memory_report()
    factor = tg.tlr_cholesky if mode == 0 else tg.tlr_ldlt

    for _ in range(args.warmup):
        F = factor(A0.copy(), cfg)
        del F
    stats = []
    barrier(dist)
    with Clocks(local) as clk:
        for s in range(args.steps):
            # the input copy (A is overwritten by its factor) is made outside the
            # factorization's own event-timed region: value = t_device of factor()
            F = factor(A0.copy(), cfg)
            stats.append(F.stats)
            del F
    barrier(dist)
    wall = sum(s.wall for s in stats)
    dev = [s.t_device for s in stats]
    t_step = allmax(dist, sum(dev) / len(dev))
    st = stats[-1]

    # accuracy of the last factorization (untimed)
    F = factor(A0.copy(), cfg)
    resid = tg.estimate_2norm_diff(A0, F, 50, 17)
    anorm = tg.estimate_2norm(A0, 50, 1)
    rk = F.L.ranks()
    xs = np.random.default_rng(7).normal(size=n)
    bvec = tg.tlr_matvec(A0, xs)
    xsol = tg.factor_solve(F, bvec)
    bwd = float(np.linalg.norm(tg.tlr_matvec(A0, xsol) - bvec) / np.linalg.norm(bvec))
    lmem = F.L.memory_report()
    del F

    # instrumented pass: per-launch CUDA events around the grouped DMMA GEMM
    os.environ["TLRG_KTIMING"] = "1"
    F = factor(A0.copy(), cfg)
    kst = F.stats
    os.environ.pop("TLRG_KTIMING", None)
    del F

    # end-to-end through the C ABI with PINNED host buffers: upload A, factorize,
    # download L (diag + U + V in the reference's flat layout) every step
    L = tg._lib
    lib = ctx.lib
    import ctypes as C
    nb_ = (n + b - 1) // b
    rows_ = [min(b, n - i * b) for i in range(nb_)]
    rks = np.ascontiguousarray(A0.ranks(), dtype=np.int32)

    def flat_sizes(rk):
        nd = sum(r * r for r in rows_)
        nu = nv = 0
        t = 0
        for i in range(1, nb_):
            for j in range(i):
                nu += rows_[i] * int(rk[t])
                nv += rows_[j] * int(rk[t])
                t += 1
        return nd, nu, nv

    def pinned(count):
        ptr = lib.tlrg_host_alloc(max(count, 1) * 8)
        assert ptr, "tlrg_host_alloc failed"
        arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(max(count, 1),))
        return ptr, arr

    nd, nu, nv = flat_sizes(rks)
    bufs = [pinned(nd), pinned(nu), pinned(nv)]
    stt = L.StatusC()
    rc = lib.tlrg_matrix_download(A0.h, bufs[0][1].ctypes.data_as(L.dp),
                                  bufs[1][1].ctypes.data_as(L.dp),
                                  bufs[2][1].ctypes.data_as(L.dp), C.byref(stt))
    assert rc == 0, stt.msg
    F = factor(A0.copy(), cfg)
    lnd, lnu, lnv = flat_sizes(F.L.ranks())
    del F
    obufs = [pinned(lnd), pinned(int(lnu * 1.05) + 4096), pinned(int(lnv * 1.05) + 4096)]
    h2d = (nd + nu + nv) * 8 + rks.nbytes
    e2e_steps = max(1, min(args.steps, 3))
    e2e_t, d2h = [], 0
    for s in range(e2e_steps):
        barrier(dist)
        t0 = time.perf_counter()
        h = C.c_void_p()
        rc = lib.tlrg_matrix_upload(ctx.h, n, b, eps, bufs[0][1].ctypes.data_as(L.dp),
                                    rks.ctypes.data_as(L.ip), bufs[1][1].ctypes.data_as(L.dp),
                                    bufs[2][1].ctypes.data_as(L.dp), C.byref(h), C.byref(stt))
        assert rc == 0, stt.msg
        Fm = factor(tg.TlrMatrix(h, ctx), cfg)
        lh = lib.tlrg_factor_L(Fm.h)
        rc = lib.tlrg_matrix_download(lh, obufs[0][1].ctypes.data_as(L.dp),
                                      obufs[1][1].ctypes.data_as(L.dp),
                                      obufs[2][1].ctypes.data_as(L.dp), C.byref(stt))
        assert rc == 0, stt.msg
        e2e_t.append(time.perf_counter() - t0)
        lnd, lnu, lnv = flat_sizes(Fm.L.ranks())
        d2h = (lnd + lnu + lnv) * 8
        del Fm
    e2e = allmax(dist, statistics.mean(e2e_t))
    for ptr, _ in bufs + obufs:
        lib.tlrg_host_free(ptr)

    peak = measure_fp64_peak() if rank == 0 else None
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            dt, cores, wall_ref = cpu_baseline_sample()
            cpu = {"value": round(dt, 3), "unit": "s", "cores": cores, "kind": "reference",
                   "sample": CPU_SAMPLE}
        except Exception as e:  # the checker is optional on the box
            cpu = {"value": None, "unit": "s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
    if rank != 0:
        return
    ach = kst.kt_gemm_flops / kst.kt_gemm_seconds / 1e12 if kst.kt_gemm_seconds else None
    line = {
        "metric": METRIC,
        "value": round(t_step, 4),
        "unit": "s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_step * 1e3, 2),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference grid points, kd-ordered; A built on device, seed 12345)",
        "config": {"workload": workload_name(args.config), "n": n, "tile": b, "eps": eps,
                   "block_samples": bs,
                   "parallelism": (f"intra-column tile split over {ws} GPUs (NCCL panel "
                                   f"all-gather per column)" if ws > 1 else "1 GPU"),
                   "l2": "inputs (A = %.2f GB) larger than L2" % (mem["total_bytes"] / 1e9)},
        "tflops_exec": round(st.flops_exec / t_step / 1e12, 3),
        "tflops_ref_equiv": round(st.flops_gemm_ref / t_step / 1e12, 3),
        "flops_exec": st.flops_exec,
        "flops_gemm_ref": st.flops_gemm_ref,
        "phases_s": {k: round(getattr(st, k), 4) for k in
                     ["t_dense", "t_misc", "t_compensation", "t_sampling", "t_orthog",
                      "t_projection", "t_recompress"]},
        "host_wall_per_step_s": round(wall / args.steps, 4),
        "e2e": {"value": round(e2e, 4), "unit": "s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(st.kernel_launches) * args.steps,
        "roofline": {"bound": "tensor",
                     "kernel": "ara_fused_kernel (FP64 DMMA; one CTA per tile, all ARA rounds + "
                               "exit projection + SVD recompression per launch)",
                     "achieved": round(st.flops_ara_kernel / st.t_ara_kernel / 1e12, 4)
                     if st.t_ara_kernel else None,
                     "peak": round(peak, 3) if peak else None, "unit": "TFLOP/s",
                     "peak_source": "measured cuBLAS DGEMM 8192^3 in this run (MEASURED_PEAKS.json "
                                    "has no FP64 entry)",
                     "frac": round(st.flops_ara_kernel / st.t_ara_kernel / 1e12 / peak, 5)
                     if st.t_ara_kernel and peak else None,
                     "traffic": ncu_traffic(),
                     "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of one "
                                       "ara_fused_kernel launch (cfg2 column 110), "
                                       "profiles/r01h_fused_ncu.txt",
                     "kernel_share_of_step": round(st.t_ara_kernel / st.t_device, 4)
                     if st.t_device else None,
                     "algorithmic_flops_per_factorization": st.flops_ara_kernel,
                     "launches_per_factorization": int(st.ara_kernel_launches),
                     "grouped_gemm": {"achieved": round(ach, 3) if ach else None,
                                      "share_of_step": round(kst.kt_gemm_seconds / kst.t_device, 4)
                                      if kst.t_device else None}},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "accuracy": {"resid_2norm": resid, "resid_rel": resid / anorm, "backward_err": bwd,
                     "L_rank_mean": float(rk.mean()), "L_rank_max": int(rk.max()),
                     "L_lowrank_bytes": int(lmem["low_rank_bytes"]),
                     "tile_rounds": int(st.tile_rounds_resident)},
        "build_s": round(t_build, 3),
    }
    print(json.dumps(line), flush=True)


def run_reference(args):
    """The unmodified reference (oracle/_ref) on the same workload, all host
    threads, rank 0 only."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import ref
    kind, n, b, eps, bs, kern, ell, nug, mode = CONFIGS[args.config]
    ref.lib()
    pts = problem_points(args.config)
    t0 = time.perf_counter()
    A = ref.build(pts, kern, ell, nug, b, eps, 0, bs, SEED)
    t_build = time.perf_counter() - t0
    times = []
    budget = float(os.environ.get("TLRG_REF_BUDGET_S", "300"))
    t_start = time.perf_counter()
    for s in range(max(1, args.steps)):
        t0 = time.perf_counter()
        F = ref.factor(A, mode, bs=bs, eps=eps, seed=SEED)
        times.append(time.perf_counter() - t0)
        del F
        if time.perf_counter() - t_start + times[-1] > budget:
            break
    v = statistics.mean(times)
    cores = ref.lib().ref_max_threads()
    line = {
        "metric": METRIC, "value": round(v, 3), "unit": "s", "n_gpus": ws,
        "steps": len(times), "warmup": 0, "ms_per_step": round(v * 1e3, 1),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference grid points, kd-ordered; A built by the reference)",
        "config": {"workload": workload_name(args.config), "n": n, "tile": b, "eps": eps,
                   "block_samples": bs, "parallelism": f"OpenMP x{cores} (host)"},
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 3), "unit": "s", "cores": cores, "kind": "reference",
                         "sample": f"full {args.config} tlr_cholesky per step "
                                   f"({len(times)} of {args.steps} steps within {budget:.0f}s)"},
        "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "build_s": round(t_build, 2),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tlrg", choices=["tlrg", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_tlrg(args)


if __name__ == "__main__":
    main()
