#!/usr/bin/env python
"""bench.py — TLR Cholesky / LDL^T time-to-solution on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tlrg|reference]
                    [--config cfg1|cfg2|cfg3|cfg4|cfg5] [--check] [--no-cpu-baseline]

Default: config 2 (the headline).  A step is one full TLR Cholesky
factorization (tlr_cholesky, factor.cpp:290-293) of the 2D exponential
covariance matrix N = 131,072, tile m = 512, eps = 1e-2, bs = 16, root seed
12345, built on the device from the reference's synthetic grid
points.  Inputs (1.17 GB) exceed L2, so no flush is needed between steps.
Configs 1, 3 and 4 are the other BASELINE.json factorizations (config 3 is
TLR LDL^T); config 5 is the batched-ARA microbench (chol_ara_update over 4,096
synthetic 512 x 512 tiles of rank 8-128, eps sweep 1e-2 .. 1e-8;
paper_2108_11932_b200/workloads.py).

value  : time-to-solution (s) per factorization (cfg5: per eps sweep),
         CUDA-event timed on the library stream, max over ranks, inputs
         resident in HBM.
e2e    : the same through the C ABI with host buffers: upload A, factorize,
         download L, per step.
accuracy: the north-star gates, computed the same way
         for both arms: ||A - LL^T||_F/||A||_F (64-probe Hutchinson, exact
         ||A||_F), ||A - LL^T||_2 (power iteration), backward and forward solve
         error, rank distribution of L.
--check: ALSO factor the reference-built A of the same config with the
         reference (oracle/_ref) and with this library, and report both accuracy
         blocks side by side (slow: the reference runs on the host).
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
    "cfg5": (None, 4096 * 512, 512, None, 32, None, None, None, None),
}
CFG5_EPS = (1e-2, 1e-4, 1e-6, 1e-8)
CFG5_TILES = 4096
SEED = 12345
# bounded reference samples of each workload for the GPU arm's cpu_baseline
CPU_SAMPLES = {
    "cfg1": ("cfg1", 16384, "full cfg1 tlr_cholesky"),
    "cfg2": ("cfg2", 32768, "cfg2 family at N=32,768 (nb=64, m=512, eps=1e-2): full reference "
                            "tlr_cholesky"),
    "cfg3": ("cfg3", 16384, "cfg3 family at N=16,384 (nb=32, m=512, eps=1e-4, bs=32): full "
                            "reference tlr_ldlt"),
    "cfg4": ("cfg4", 32768, "cfg4 family at N=32,768 (nb=32, m=1024, eps=1e-3, bs=32): full "
                            "reference tlr_cholesky"),
    "cfg5": ("cfg5", 256, "256 of the 4,096 cfg5 tiles, full eps sweep, reference "
                          "chol_ara_update"),
}
FP64_NOMINAL = 148 * 128 * 1.965e9 / 1e12  # 64 DFMA/clk/SM x 148 SMs at 1965 MHz


def workload_name(cfg):
    if cfg == "cfg5":
        return (f"batched ARA microbench: {CFG5_TILES} synthetic 512x512 tiles of rank 8-128, "
                f"chol_ara_update(k=0), bs=32, eps sweep 1e-2..1e-8 (cfg5)")
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


# per-launch DRAM traffic of the dominant kernel from this round's committed
# ncu --set full capture of that config (null when none was taken)
NCU_TRAFFIC = {
    "cfg2": "profiles/r02_cfg2_fused_ncu.txt",
}


def ncu_traffic(cfg):
    path = NCU_TRAFFIC.get(cfg)
    if not path:
        return None, None
    try:
        tot = 0
        for line in open(os.path.join(ROOT, path)):
            if line.startswith(("dram__bytes_read.sum:", "dram__bytes_write.sum:")):
                tot += int(float(line.split(":")[1].split()[0]))
        return (tot or None), path
    except OSError:
        return None, None


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
    """cuBLAS DGEMM 8192^3 via torch (burst, best of 5): the FP64 roofline
    denominator (MEASURED_PEAKS.json carries HBM and bf16 only)."""
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


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback 6.65 TB/s"


def problem_points(cfg, n=None):
    from paper_2108_11932_b200 import geometry as G
    kind, n0, b = CONFIGS[cfg][:3]
    return G.kd_order(G.generate_points(kind, n or n0, 0), b).matrix_order()


def round6(d):
    return {k: (round(v, 9) if isinstance(v, float) else v) for k, v in d.items()}


# ----------------------------------------------------------------- CPU legs --
def cpu_baseline_sample(cfg):
    """The reference (oracle/_ref, unmodified sources) on a bounded sample of
    the same workload, all host threads."""
    from oracle import ref
    ref.lib()
    name, n, what = CPU_SAMPLES[cfg]
    if cfg == "cfg5":
        from paper_2108_11932_b200 import workloads as W
        nn, b, ranks, U, V = W.cfg5_column(n)
        A = ref.matrix_from_flat(nn, b, 1e-2, None, ranks, U, V)
        t = time.perf_counter()
        for eps in CFG5_EPS:
            ref.chol_ara_update(A, 0, bs=32, eps=eps, seed=SEED)
        dt = time.perf_counter() - t
        return dt, ref.lib().ref_max_threads(), what
    kind, _, b, eps, bs, kern, ell, nug, mode = CONFIGS[cfg]
    pts = problem_points(cfg, n)
    A = ref.build(pts, kern, ell, nug, b, eps, 0, bs, SEED)
    t = time.perf_counter()
    ref.factor(A, mode, bs=bs, eps=eps, seed=SEED)
    dt = time.perf_counter() - t
    return dt, ref.lib().ref_max_threads(), what


# --------------------------------------------------------------- GPU arm ----
def run_tlrg(args):
    if args.config == "cfg5":
        return run_tlrg_cfg5(args)
    ws, rank, local = dist_env()
    dist = dist_init(ws, "nccl")
    import numpy as np

    import paper_2108_11932_b200 as tg
    from paper_2108_11932_b200.tlr import accuracy, build_tlr
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

    # accuracy of one more factorization (untimed)
    F = factor(A0.copy(), cfg)
    acc = accuracy(A0, F)
    acc["tile_rounds"] = int(F.stats.tile_rounds_resident)
    del F

    # instrumented pass: per-launch CUDA events around the grouped DMMA GEMM
    os.environ["TLRG_KTIMING"] = "1"
    F = factor(A0.copy(), cfg)
    kst = F.stats
    os.environ.pop("TLRG_KTIMING", None)
    del F

    e2e, h2d, d2h = e2e_factor(args, ctx, A0, factor, cfg, n, b, eps, dist)

    peak = measure_fp64_peak() if rank == 0 else None
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            dt, cores, what = cpu_baseline_sample(args.config)
            cpu = {"value": round(dt, 3), "unit": "s", "cores": cores, "kind": "reference",
                   "sample": what}
        except Exception as e:  # the checker is optional on the box
            cpu = {"value": None, "unit": "s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
    check = run_check(args, ctx, factor, cfg) if (args.check and rank == 0) else None
    if rank != 0:
        return
    ach = kst.kt_gemm_flops / kst.kt_gemm_seconds / 1e12 if kst.kt_gemm_seconds else None
    traffic, tsrc = ncu_traffic(args.config)
    fused = st.t_ara_kernel > 0
    if fused:
        r_ach = st.flops_ara_kernel / st.t_ara_kernel / 1e12
        roof = {"bound": "tensor",
                "kernel": "ara_fused_kernel (FP64 DMMA; one CTA per tile, all ARA rounds + "
                          "exit projection + SVD recompression per launch)",
                "achieved": round(r_ach, 4),
                "algorithmic_flops_per_factorization": st.flops_ara_kernel,
                "launches_per_factorization": int(st.ara_kernel_launches),
                "kernel_share_of_step": round(st.t_ara_kernel / st.t_device, 4)}
    else:
        # graph path (bs = 32): the ARA phases as a whole, reference formulation
        t_ara = st.t_sampling + st.t_projection + st.t_recompress
        r_ach = st.flops_gemm_ref / t_step / 1e12
        roof = {"bound": "tensor",
                "kernel": "whole factorization, reference-formulation F_gemm (graph-path ARA: "
                          "grouped DMMA GEMMs + panel MGS + batched Jacobi)",
                "achieved": round(r_ach, 4), "ara_phase_seconds": round(t_ara, 4)}
    roof.update({"peak": round(peak, 3) if peak else None, "unit": "TFLOP/s",
                 "peak_source": "measured cuBLAS DGEMM 8192^3 in this run (MEASURED_PEAKS.json "
                                "has no FP64 entry); nominal %.1f" % FP64_NOMINAL,
                 "frac": round(r_ach / peak, 5) if peak else None,
                 "traffic": traffic, "traffic_source": tsrc,
                 "grouped_gemm": {"achieved": round(ach, 3) if ach else None,
                                  "share_of_step": round(kst.kt_gemm_seconds / kst.t_device, 4)
                                  if kst.t_device else None}})
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
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "accuracy": round6(acc),
        "build_s": round(t_build, 3),
    }
    if check is not None:
        line["check"] = check
    print(json.dumps(line), flush=True)


def e2e_factor(args, ctx, A0, factor, cfg, n, b, eps, dist):
    """End to end through the C ABI with PINNED host buffers: upload A,
    factorize, download L (diag + U + V in the reference's flat layout)."""
    import ctypes as C

    import numpy as np

    import paper_2108_11932_b200 as tg
    L = tg._lib
    lib = ctx.lib
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
    return e2e, h2d, d2h


def run_check(args, ctx, factor, cfg):
    """Same-A parity: the reference builds A on the host; the reference and
    this library factor THAT matrix; both accuracy blocks side by side."""
    from oracle import ref

    import paper_2108_11932_b200 as tg
    from paper_2108_11932_b200.tlr import accuracy
    kind, n, b, eps, bs, kern, ell, nug, mode = CONFIGS[args.config]
    t0 = time.perf_counter()
    Ar = ref.build(problem_points(args.config), kern, ell, nug, b, eps, 0, bs, SEED)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    Fr = ref.factor(Ar, mode, bs=bs, eps=eps, seed=SEED)
    t_ref = time.perf_counter() - t0
    acc_ref = ref.accuracy(Ar, Fr)
    diag, ranks, U, V = Ar.to_flat()
    Ag = tg.TlrMatrix.from_flat(n, b, eps, diag, ranks, U, V, ctx=ctx)
    F = factor(Ag.copy(), cfg)
    acc_gpu = accuracy(Ag, F)
    same_tiles = float((F.L.ranks() == Fr.L_ranks()).mean())
    return {"A": "reference-built (oracle/_ref build_tlr, seed 12345), uploaded unchanged",
            "reference": round6(acc_ref), "tlrg": round6(acc_gpu),
            "tiles_with_equal_rank": same_tiles, "ref_factor_s": round(t_ref, 2),
            "ref_build_s": round(t_build, 2), "tlrg_factor_s": round(F.stats.t_device, 4)}


def run_tlrg_cfg5(args):
    """Config 5: chol_ara_update(k = 0) over the synthetic column (the
    reference's batched-ARA entry point, ara.cpp:302-419) per eps."""
    ws, rank, local = dist_env()
    dist = dist_init(ws, "nccl")
    import ctypes as C

    import numpy as np

    import paper_2108_11932_b200 as tg
    from paper_2108_11932_b200 import workloads as W
    from paper_2108_11932_b200.util import rank_summary
    ctx = tg.Context(local)
    n, b, ranks, U, V = W.cfg5_column(CFG5_TILES)
    A = tg.TlrMatrix.from_flat(n, b, 1e-2, None, ranks, U, V, ctx=ctx)
    per_eps, acc = {}, {}
    with Clocks(local) as clk:
        for eps in CFG5_EPS:
            cfg = tg.AraConfig(block_samples=32, eps=eps, seed=SEED)
            for _ in range(args.warmup):
                tg.chol_ara_update(A, None, 0, cfg)
            ts, st = [], {}
            for _ in range(args.steps):
                st = {}
                res = tg.chol_ara_update(A, None, 0, cfg, stats=st)
                ts.append(st["t_device"])
            per_eps[f"{eps:g}"] = {"s": round(statistics.mean(ts), 4),
                                   "tile_rounds": st["tile_rounds"],
                                   "flops_ref": st["flops_ref"]}
            rk = [r.Q.shape[1] for r in res]
            # relative approximation error of every tile, worst case (spot check
            # of 64 tiles against the stored factors)
            worst = 0.0
            for r in res[:: max(1, len(res) // 64)]:
                t = r.i - 1
                rt = int(ranks[r.i * (r.i - 1) // 2])
                off = sum(int(ranks[(j + 1) * j // 2]) for j in range(t)) * b
                Ut = U[off:off + b * rt].reshape(rt, b).T
                Vt = V[off:off + b * rt].reshape(rt, b).T
                err = np.linalg.norm(Ut @ Vt.T - r.Q @ r.B.T, 2)
                worst = max(worst, err / eps)
            acc[f"{eps:g}"] = dict(rank_summary(rk), worst_err_over_eps=worst)
    t_step = allmax(dist, sum(v["s"] for v in per_eps.values()))
    flops = sum(v["flops_ref"] for v in per_eps.values())
    # e2e: host flat arrays (pinned) -> upload -> chol_ara_update -> results to host
    lib = ctx.lib
    L = tg._lib

    def pinned_copy(a):
        ptr = lib.tlrg_host_alloc(max(a.nbytes, 8))
        arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(max(a.size, 1),))
        arr[:a.size] = a
        return ptr, arr
    pU, pV = pinned_copy(U), pinned_copy(V)
    e2e_t = []
    d2h = 0
    for _ in range(max(1, min(args.steps, 2))):
        t0 = time.perf_counter()
        h = C.c_void_p()
        stt = L.StatusC()
        rc = lib.tlrg_matrix_upload(ctx.h, n, b, 1e-2, None, ranks.ctypes.data_as(L.ip),
                                    pU[1].ctypes.data_as(L.dp), pV[1].ctypes.data_as(L.dp),
                                    C.byref(h), C.byref(stt))
        assert rc == 0, stt.msg
        Am = tg.TlrMatrix(h, ctx)
        d2h = 0
        for eps in CFG5_EPS:
            res = tg.chol_ara_update(Am, None, 0, tg.AraConfig(block_samples=32, eps=eps,
                                                                 seed=SEED))
            d2h += sum((r.Q.size + r.B.size) * 8 for r in res)
        e2e_t.append(time.perf_counter() - t0)
        del Am
    for p, _ in (pU, pV):
        lib.tlrg_host_free(p)
    e2e = allmax(dist, statistics.mean(e2e_t))
    peak = measure_fp64_peak() if rank == 0 else None
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            dt, cores, what = cpu_baseline_sample("cfg5")
            cpu = {"value": round(dt, 3), "unit": "s", "cores": cores, "kind": "reference",
                   "sample": what}
        except Exception as e:
            cpu = {"value": None, "unit": "s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
    if rank != 0:
        return
    ach = flops / t_step / 1e12
    line = {
        "metric": "batched ARA time (s) per eps sweep, 4,096 variable-rank 512x512 tiles",
        "value": round(t_step, 4), "unit": "s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 2), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (workloads.cfg5_column, seed 4242)",
        "config": {"workload": workload_name("cfg5"), "tiles": CFG5_TILES, "tile": b,
                   "block_samples": 32, "eps": list(CFG5_EPS), "parallelism": "1 GPU",
                   "l2": "inputs (U+V = %.2f GB) larger than L2" % ((U.nbytes + V.nbytes) / 1e9)},
        "per_eps": per_eps,
        "e2e": {"value": round(e2e, 4), "unit": "s", "h2d_bytes_per_step": int(U.nbytes + V.nbytes
                                                                             + ranks.nbytes),
                "d2h_bytes_per_step": int(d2h)},
        "roofline": {"bound": "tensor", "kernel": "batched ARA (sampling + projection, "
                                                  "reference-formulation flops)",
                     "achieved": round(ach, 4), "peak": round(peak, 3) if peak else None,
                     "unit": "TFLOP/s", "frac": round(ach / peak, 5) if peak else None,
                     "peak_source": "measured cuBLAS DGEMM 8192^3 in this run",
                     "traffic": None},
        "cpu_baseline": cpu, "clocks": clk.summary(), "accuracy": acc,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------- reference arm ---
def run_reference(args):
    """The unmodified reference (oracle/_ref) on the same workload, all host
    threads, rank 0 only."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import ref
    ref.lib()
    cores = ref.lib().ref_max_threads()
    budget = float(os.environ.get("TLRG_REF_BUDGET_S", "300"))
    if args.config == "cfg5":
        from paper_2108_11932_b200 import workloads as W
        from paper_2108_11932_b200.util import rank_summary
        n, b, ranks, U, V = W.cfg5_column(CFG5_TILES)
        A = ref.matrix_from_flat(n, b, 1e-2, None, ranks, U, V)
        times, acc = [], {}
        t_start = time.perf_counter()
        for s in range(max(1, args.steps)):
            t0 = time.perf_counter()
            for eps in CFG5_EPS:
                res = ref.chol_ara_update(A, 0, bs=32, eps=eps, seed=SEED)
                if s == 0:
                    acc[f"{eps:g}"] = rank_summary([r["Q"].shape[1] for r in res])
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - t_start + times[-1] > budget:
                break
        v = statistics.mean(times)
        metric = "batched ARA time (s) per eps sweep, 4,096 variable-rank 512x512 tiles"
        cfgd = {"workload": workload_name("cfg5"), "tiles": CFG5_TILES, "tile": b,
                "block_samples": 32, "eps": list(CFG5_EPS),
                "parallelism": f"OpenMP x{cores} (host)"}
        t_build = 0.0
    else:
        kind, n, b, eps, bs, kern, ell, nug, mode = CONFIGS[args.config]
        pts = problem_points(args.config)
        t0 = time.perf_counter()
        A = ref.build(pts, kern, ell, nug, b, eps, 0, bs, SEED)
        t_build = time.perf_counter() - t0
        times = []
        t_start = time.perf_counter()
        F = None
        for s in range(max(1, args.steps)):
            F = None
            t0 = time.perf_counter()
            F = ref.factor(A, mode, bs=bs, eps=eps, seed=SEED)
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - t_start + times[-1] > budget:
                break
        v = statistics.mean(times)
        acc = round6(ref.accuracy(A, F))
        metric = METRIC
        cfgd = {"workload": workload_name(args.config), "n": n, "tile": b, "eps": eps,
                "block_samples": bs, "parallelism": f"OpenMP x{cores} (host)"}
    line = {
        "metric": metric, "value": round(v, 3), "unit": "s", "n_gpus": ws,
        "steps": len(times), "warmup": 0, "ms_per_step": round(v * 1e3, 1),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference grid points, kd-ordered; A built by the reference)"
        if args.config != "cfg5" else "synthetic (workloads.cfg5_column, seed 4242)",
        "config": cfgd,
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 3), "unit": "s", "cores": cores, "kind": "reference",
                         "sample": f"full {args.config} per step "
                                   f"({len(times)} of {args.steps} steps within {budget:.0f}s)"},
        "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "accuracy": acc,
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
    ap.add_argument("--check", action="store_true",
                    help="also factor the reference-built A with both arms (slow)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_tlrg(args)


if __name__ == "__main__":
    main()
