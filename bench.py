#!/usr/bin/env python
"""bench.py — RHS·iterations/s of the simultaneous-RHS Krylov hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--method egl_qmr] [--config 3] [--m 256]

A "step" is one full iteration of the method (every §8(a) row of SURVEY.md:
SpMM A·P with the fused Gram epilogue, the A^H vector product, the fused block
updates with their reductions, the s x s device coefficient phases and the
convergence test) over config 3 of BASELINE.json (3D 7-point convection-
diffusion 256^3, n = 16.8M, 117M nnz, FP64, s = 16 Gaussian RHS from seed 2),
method eGl-QMR. Inputs are resident in HBM before the
timed region; every block is 2.1 GB, far larger than the 126 MB L2, so no L2
flush is needed between steps.

One JSON line on rank 0 with: value (whole-job RHS·it/s), e2e (the same metric
through srk_solve_host with host B/X, copies inside the timed region),
roofline (the dominant kernel: the kernel family with the largest share of the
step, its launches timed live with CUDA events inside the timed region and its
algorithmic bytes counted by the engine per SURVEY §8(d).3), roofline_spmm (the
same for the A·P SpMM with its fused Gram), iteration.kernels (every family),
cpu_baseline (the oracle on a bounded sample:
one config-3 iteration on the host cores), clocks (nvidia-smi during the
timed region), gpu_launches (kernels in the timed region).

--impl reference times the oracle (oracle/, numpy/scipy on the host cores) on
the same workload: each step is one oracle iteration, W+K of them.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "RHS·iterations/sec"
P64_TFLOPS = 37.1  # FP64 tensor-core (DMMA) peak measured by scripts/fp64_probe.cu on this B200 model
UNIT = "RHS·it/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, uuid: str | None):
        self.uuid = uuid
        self.rows = []
        self.proc = None

    def start(self):
        cmd = ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200"]
        if self.uuid:
            cmd += ["-i", self.uuid]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def oracle_iteration_rate(method, A, B, iters: int):
    """Time the oracle (as it stands) per iteration via timestamps of its A-products."""
    import scipy.sparse as sp

    import oracle
    stamps = []

    class TimedCSR(sp.csr_matrix):
        def __matmul__(self, other):
            stamps.append(time.perf_counter())
            return super().__matmul__(other)

    As = TimedCSR((A.values, A.col_idx, A.row_ptr), shape=(A.n, A.n))
    t0 = time.perf_counter()
    oracle.solve(method, As, B, tol=1e-300, maxit=iters, record=0)
    total = time.perf_counter() - t0
    per_it_products = 2 if "bicgstab" in method else 1
    # stamps: [R0, it1 (x per_it), it2, ..., final true residual]
    it_starts = stamps[1:1 + iters * per_it_products:per_it_products] + [stamps[-1]]
    durs = np.diff(it_starts)
    return durs, total


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info
        th = max((d.get("num_threads", 1) for d in threadpool_info()), default=1)
    except Exception:
        th = os.cpu_count()
    return model, th


def run_reference(args, A, B, s, cfgd, scale: float = 1.0, note: str | None = None):
    # one oracle iteration of config 3 takes ~6-10 s on the host: bound the sample
    # to <= 3 timed iterations after <= 3 warm-up iterations (the contract's W >= 3)
    # so the run ends within a few minutes
    steps, warm = min(args.steps, 3), min(args.warmup, 3)
    durs, total = oracle_iteration_rate(args.method, A, B, warm + steps)
    timed = durs[warm:warm + steps] if len(durs) >= warm + steps else durs[-steps:]
    T = float(np.sum(timed)) / scale
    value = s * len(timed) / T
    model, th = cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(timed), "warmup": warm, "ms_per_step": 1e3 * T / len(timed), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfgd,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": th, "kind": "oracle",
                         "sample": (note or f"{len(timed)} oracle iterations of {args.method} on the full workload")
                                   + f" (numpy/scipy; scipy.sparse products single-threaded), CPU {model}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--method", default=None, help="default: the config's method (cfg3 egl_qmr, cfg4 gl_bicgstab)")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--m", type=int, default=None, help="override the grid size (tests)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    import synth
    if args.method is None:
        args.method = {1: "egl_bicg", 2: "bl_bicg_rq", 3: "egl_qmr", 4: "gl_bicgstab", 5: "egl_bicg"}[args.config]
    c = synth.CONFIGS[args.config]
    bsr = None
    bsr_nnzb = 0
    if args.config == 4:
        # a0: the lattice operator in BSR-12 form with the unit diagonal implied
        # (the scalar CSR of 32^4 would be 24.4 GB and gather 18.6 KB per row)
        L = args.m or c["L"]
        bsr = synth.lattice_4d_bsr(L, c["kappa"], c["seed"])
        n = L ** 4 * 12
        B = synth.random_rhs(n, c["s"], c["seed"], True)

        class A:  # the scalar view (for the config record)
            pass
        A.n, A.nnz = n, len(bsr[1]) * 144 + n
        bsr_nnzb = len(bsr[1])
        import hashlib
        h = hashlib.sha256()
        for arr in (*bsr, B):
            h.update(np.ascontiguousarray(arr).view(np.uint8).data)
        ihash = h.hexdigest()[:16]
    else:
        A, B = synth.make_config(args.config, m=args.m)
        ihash = synth.input_hash(A, B)
    s = B.shape[1]
    esz = 16 if np.iscomplexobj(B) else 8
    cfgd = {"workload": f"{c['name']} ({'m=%d' % (args.m or c.get('m', c.get('L', 0)))}) {args.method}",
            "method": args.method, "n": A.n, "nnz": A.nnz, "s": s, "dtype": c["dtype"],
            "operator": "BSR-12, unit diagonal implied" if bsr is not None else "CSR",
            "parallelism": "replicas" if world > 1 else "single",
            "l2": ("no flush: every n x s block (%.2f GB) exceeds the 126 MB L2" % (A.n * s * esz / 1e9)
                   if A.n * s * esz > 126e6 else
                   "no flush: the whole problem (%.1f KB per block) is L2-resident by design (latency-bound)"
                   % (A.n * s * esz / 1e3)),
            "inputs_hash": ihash}

    if args.impl == "reference":
        if rank == 0:
            if bsr is not None:  # bounded sample: the oracle on the 16^4 lattice, scaled by the row ratio
                As, Bs = synth.make_config(4, m=16)
                run_reference(args, As, Bs, s, cfgd, scale=As.n / A.n,
                              note="oracle on config 4's operator at 16^4 sites (1/16 of the rows), "
                                   "per-iteration time scaled x16")
            else:
                run_reference(args, A, B, s, cfgd)
        return

    import torch
    import paper_1504_04395_b200 as srk
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", torch.cuda.current_device())
    srk.load_library()
    if world > 1 and bsr is not None:
        # config 4: the lattice's block rows split into t-slabs (contiguous lexicographic
        # site ranges, nnz-balanced); each product exchanges the 12 rows of every ghost block
        srk.init_distributed()
        boff = srk.partition_rows(bsr[0], world)
        M = srk.DistMatrix.from_bsr(*bsr, boff, rank, unit_diag=True)
        o0, o1 = int(boff[rank]) * 12, int(boff[rank + 1]) * 12
        B = np.ascontiguousarray(B[o0:o1])
        del bsr
        bsr = True
        cfgd["parallelism"] = f"t-slabs x{world} (BSR-12 block halo + NCCL allreduce)"
    elif world > 1:
        # a8: A and every n x s block row-partitioned (nnz-balanced contiguous ranges);
        # halo exchange before each SpMM (overlapped with the interior rows' product) and an
        # NCCL allreduce of every reduction
        srk.init_distributed()
        off = srk.partition_rows(A.row_ptr, world)
        M = srk.DistMatrix(A, off, rank, need_adjoint=srk.NEEDS_ADJOINT[args.method])
        o0, o1 = int(off[rank]), int(off[rank + 1])
        B = np.ascontiguousarray(B[o0:o1])
        cfgd["parallelism"] = f"row-partition x{world} (halo exchange overlapped with the interior rows + NCCL allreduce)"
    elif bsr is not None:
        M = srk.Matrix.from_bsr(*bsr, unit_diag=True)
        del bsr
    else:
        M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[args.method])
    n_local = B.shape[0]
    Bd = torch.from_numpy(B).to(dev)
    K, W = args.steps, args.warmup

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    # ---- device-resident timed region
    # config 1 is latency-bound: its step runs as the product does,
    # W-iteration CUDA graphs replayed between polls (captured in the warm-up), and
    # without per-launch events (which would serialise it); no roofline fraction
    latency = args.config == 1
    poll = W if latency else W + K + 1
    warm = 2 * W if latency else W
    REPEATS = 5  # the median of 5 timed windows is reported beside the first
    sv = srk.Solver(M, s, args.method, tol=1e-300, maxit=warm + REPEATS * K + 1, poll_every=poll,
                    check_true_residual=False)
    sv.start(Bd)
    sv.iterate(W)
    if latency:
        sv.iterate(W)  # captures the graph
    l0 = sv.report().kernel_launches
    uuid = None
    try:
        uuid = str(torch.cuda.get_device_properties(dev).uuid)
        uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
    except Exception:
        pass
    clk = ClockSampler(uuid)
    barrier()
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sv.profile(not latency)
    e0.record()
    st = sv.iterate(K)
    e1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    recs = sv.profile_launches()
    rep = sv.report()
    launches = rep.kernel_launches - l0
    assert st == 0 and rep.iterations == warm + K, (st, rep)
    # four more windows of exactly K steps (same solver, no profiling), for the median of 5
    windows = [ms]
    for _ in range(REPEATS - 1):
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        sv.iterate(K)
        f1.record()
        torch.cuda.synchronize()
        windows.append(f0.elapsed_time(f1))
    if world > 1:
        t = torch.tensor(windows, device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        windows = [float(x) for x in t.tolist()]
        ms = windows[0]
    value = s * K / (ms / 1e3)  # the whole job iterates the same s right-hand sides
    med = statistics.median(windows)
    median5 = {"value": s * K / (med / 1e3), "ms_per_step": med / K,
               "windows_ms_per_step": [w / K for w in windows],
               "note": "median of 5 timed windows of K steps (SURVEY §8(d).4); the first window is `value`, "
                       "timed with per-launch events (the profile of `roofline`), the other four without"}

    # ---- rooflines, timed live: every launch of the timed region carries its
    # algorithmic bytes (computed by the engine); launches are
    # grouped into kernel families, and `roofline` reports the family with the
    # largest share of the step (the dominant kernel)
    peak, peak_src = peaks()
    fams = {}
    for tag, sig, t_ms, nb in recs:
        if tag in ("spmm", "spmm_adj"):
            name = f"{tag} s={sig}"
        elif tag == "update":
            name = f"update {sig // 16} in / {sig % 16} out"
        else:
            name = tag
        key = (name, round(nb))
        f = fams.setdefault(key, {"kernel": name, "ms_total": 0.0, "launches": 0, "bytes_per_launch": nb})
        f["ms_total"] += t_ms
        f["launches"] += 1
    kern = []
    for f in fams.values():
        avg = f["ms_total"] / f["launches"] / 1e3
        ach = f["bytes_per_launch"] / avg / 1e9 if f["bytes_per_launch"] > 0 else None
        kern.append({"kernel": f["kernel"], "launches": f["launches"], "avg_launch_ms": avg * 1e3,
                     "algorithmic_bytes_per_launch": f["bytes_per_launch"], "achieved_gbs": ach,
                     "frac": (ach / peak) if ach else None, "share_of_step": f["ms_total"] / ms})
    kern.sort(key=lambda k: -k["share_of_step"])
    dom = next((k for k in kern if k["achieved_gbs"]), None)
    spm = next((k for k in kern if k["kernel"].startswith("spmm s=")), None)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        traffic = tj.get(f"cfg{args.config}_{args.method}_" + ("spmm" if dom is spm else "dominant"))
    if dom is None:  # latency-bound config 1: the whole problem sits in L2
        roof = {"bound": "latency", "achieved": None, "peak": None, "unit": "GB/s", "frac": None, "traffic": None,
                "note": "config 1 (n = 1024) is latency-bound (SURVEY §8(d).2): RHS·it/s only; "
                        "step = W-iteration CUDA graph replays"}
    else:
        roof = {"bound": "hbm", "achieved": dom["achieved_gbs"], "peak": peak, "unit": "GB/s",
                "frac": dom["achieved_gbs"] / peak, "traffic": traffic, "kernel": dom["kernel"],
                "algorithmic_bytes_per_launch": dom["algorithmic_bytes_per_launch"],
                "avg_launch_ms": dom["avg_launch_ms"], "launches": dom["launches"],
                "share_of_step": dom["share_of_step"], "peak_source": peak_src}
    if bsr_nnzb and spm:
        # config 4's BSR-12 product sits near the FP64 ridge: its bound is
        # max(bytes / BW, flops / P64); useful flops = 8 real flops per complex multiply-add,
        # 144 entries per block, s columns (the implied identity is not counted)
        fl = bsr_nnzb * 144 * 8 * s
        t_mem = spm["algorithmic_bytes_per_launch"] / (peak * 1e9)
        t_fl = fl / (P64_TFLOPS * 1e12)
        t_act = spm["avg_launch_ms"] / 1e3
        spm["flops_per_launch"] = fl
        spm["achieved_tflops"] = fl / t_act / 1e12
        spm["bound"] = "fp64" if t_fl > t_mem else "hbm"
        spm["frac_of_bound"] = max(t_mem, t_fl) / t_act
        spm["p64_tflops"] = P64_TFLOPS
        spm["p64_source"] = "measured DMMA peak of this B200 model (scripts/fp64_probe.cu, DESIGN.md §7)"
    it_bytes = sum(nb for _, _, _, nb in recs) / K
    breakdown = {}
    for tag, _, t_ms, _ in recs:
        e = breakdown.setdefault(tag, {"ms_total": 0.0, "launches": 0})
        e["ms_total"] += t_ms
        e["launches"] += 1

    # ---- end to end through the C-ABI with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        Bh = torch.from_numpy(B).pin_memory()
        Xh = torch.zeros_like(Bh).pin_memory()
        # untimed warm-up call: the context keeps the solver workspace and the staging
        # blocks for the next call with the same operator / width / method / options
        srk.solve_host(M, Bh.numpy(), args.method, tol=1e-300, maxit=K, X0=Xh.numpy(), poll_every=K + 1, inplace=True,
                       x0_zero=True)
        barrier()
        t0 = time.perf_counter()
        X, r2 = srk.solve_host(M, Bh.numpy(), args.method, tol=1e-300, maxit=K, X0=Xh.numpy(), poll_every=K + 1,
                               inplace=True, x0_zero=True)  # X0 = 0: X is output only
        T = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([T], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            T = float(t.item())
        nbytes = B.nbytes
        e2e = {"value": s * r2.iterations / T, "unit": UNIT, "h2d_bytes_per_step": nbytes / K,
               "d2h_bytes_per_step": nbytes / K,
               "note": "srk_solve_host (after one untimed call that sizes the cached workspace), X0 = 0 (P:639): "
                       "H2D of B, R0 = B, K iterations, the final true residual, D2H of X"}

    # ---- end to end, full solve: B on the host to the converged X on the host (tol 1e-8)
    e2e_full = None
    if not args.no_e2e and world == 1 and not latency:
        Bh = torch.from_numpy(B).pin_memory()
        Xh = torch.zeros_like(Bh).pin_memory()
        srk.solve_host(M, Bh.numpy(), args.method, tol=1e-8, maxit=2000, X0=Xh.numpy(), inplace=True, x0_zero=True)
        barrier()
        t0 = time.perf_counter()
        X, r3 = srk.solve_host(M, Bh.numpy(), args.method, tol=1e-8, maxit=2000, X0=Xh.numpy(), inplace=True,
                               x0_zero=True)
        T = time.perf_counter() - t0
        e2e_full = {"value": s * r3.iterations / T, "unit": UNIT, "seconds": T, "iterations": r3.iterations,
                    "outcome": r3.outcome, "final_true_rel_residual": r3.final_true_rel_residual,
                    "h2d_bytes": B.nbytes, "d2h_bytes": B.nbytes,
                    "note": "srk_solve_host to convergence (tol 1e-8, maxit 2000, X0 = 0), host buffers, "
                            "after one untimed identical call (workspace sizing)"}

    # ---- CPU baseline: the oracle on one config-3 iteration (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        model, th = cpu_info()
        if args.config == 4:  # bounded sample: the 16^4 lattice (1/16 of the rows), time scaled x16
            As, Bs = synth.make_config(4, m=16)
            durs, total = oracle_iteration_rate(args.method, As, Bs, 2)
            t_it = float(durs[-1]) * A.n / As.n
            cpu = {"value": s / t_it, "unit": UNIT, "cores": th, "kind": "oracle",
                   "sample": f"iteration 2 of {args.method} on config 4's operator at 16^4 sites "
                             f"({durs[-1]:.1f} s), scaled by the row ratio x{A.n // As.n}, CPU {model}"}
        else:
            durs, total = oracle_iteration_rate(args.method, A, B, 2)
            cpu = {"value": s / float(durs[-1]), "unit": UNIT, "cores": th, "kind": "oracle",
                   "sample": f"iteration 2 of {args.method} on the full config-{args.config} workload "
                             f"({durs[-1]:.1f} s; oracle call {total:.1f} s incl. setup), CPU {model}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if esz == 8 else "c128", "data": "synthetic", "config": cfgd,
            "roofline": roof, "roofline_spmm": spm, "cpu_baseline": cpu, "e2e": e2e, "e2e_full_solve": e2e_full,
            "median_of_5": median5,
            "gpu_launches": int(launches), "clocks": clocks,
            "iteration": {"algorithmic_bytes": it_bytes or None,
                          "achieved_gbs": (it_bytes / (ms / K / 1e3) / 1e9) if it_bytes else None,
                          "frac_of_peak": (it_bytes / (ms / K / 1e3) / 1e9 / peak) if it_bytes else None,
                          "kernels": kern, "by_tag": breakdown},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
