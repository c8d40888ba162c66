"""BSR-12 product timing on config 4's lattice (32^4 sites, 12 complex dof, s = 12): the
M = 24 / K = 12 tensor-core form (bsr12_kernel2) against the padded form (SRK_BSR_OLD=1, read per
launch), alone and with the fused trace operand; CUDA events on the library's stream, median of 10.
Prints ms, algorithmic GB/s and useful FP64 TFLOP/s (2 * 4 * 12 * 12 * s flops per block).
    python scripts/bsr_probe.py [L] [reps]
"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1504_04395_b200 as srk  # noqa: E402
import synth  # noqa: E402


def med_ms(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    srk.load_library()
    t0 = time.time()
    brp, bcol, blocks = synth.lattice_4d_bsr(L)
    print(f"lattice {L}^4 generated in {time.time() - t0:.0f} s", flush=True)
    M = srk.Matrix.from_bsr(brp, bcol, blocks, unit_diag=True)
    del blocks
    nb, s = L ** 4, 12
    n = nb * 12
    P = torch.from_numpy(synth.random_rhs(n, s, 3, True)).cuda()
    Y = torch.from_numpy(synth.random_rhs(n, s, 5, True)).cuda()
    Q = torch.empty_like(P)
    abytes = (nb + 1) * 4 + 8 * nb * (4 + 2304) + 2 * n * s * 16
    flops = 8.0 * nb * 8 * 12 * 12 * s
    ref0 = None
    for cfg in [int(x) for x in os.environ.get("BSR_CFGS", "0,1,2,3,4,5").split(",")]:
        os.environ["SRK_BSR_CFG"] = str(cfg)   # (warps per CTA, ring stages, epilogue staging): see bsr.cu launch_s
        t = med_ms(lambda: srk.spmm_block(M, P, Q=Q), reps)
        q = Q.clone()
        tt = med_ms(lambda: srk.spmm_block(M, P, gram="trace", Y=Y, Q=Q), reps)
        ref0 = q if ref0 is None else ref0
        print(f"launch cfg {cfg}: {t:.3f} ms  {abytes / t / 1e6:.0f} GB/s  {flops / t / 1e9:.1f} TFLOP/s | with trace operand {tt:.3f} ms"
              f" | bitwise equal to cfg 0: {bool(torch.equal(q, ref0))}", flush=True)
    os.environ.pop("SRK_BSR_CFG", None)
    for w in [int(x) for x in os.environ.get("BSR_TILES", "0,4").split(",")]:
        M.set_row_order(synth.lattice_tile_order(L, w) if w else None)
        t = med_ms(lambda: srk.spmm_block(M, P, Q=Q), reps)
        tt = med_ms(lambda: srk.spmm_block(M, P, gram="trace", Y=Y, Q=Q), reps)
        print(f"z-tile {w:2d} planes (0 = natural order): {t:.3f} ms  {abytes / t / 1e6:.0f} GB/s  {flops / t / 1e9:.1f} TFLOP/s"
              f" | with trace operand {tt:.3f} ms", flush=True)
    M.set_row_order(None)
    if os.environ.get("BSR_TILES_ONLY"):
        return
    ref = None
    for old in (0, 1, 0, 1):
        if old:
            os.environ["SRK_BSR_OLD"] = "1"
        else:
            os.environ.pop("SRK_BSR_OLD", None)
        t = med_ms(lambda: srk.spmm_block(M, P, Q=Q), reps)
        q = Q.clone()
        tt = med_ms(lambda: srk.spmm_block(M, P, gram="trace", Y=Y, Q=Q), reps)
        if ref is None:
            ref = q
        dev = float((q - ref).abs().max() / ref.abs().max())
        print(f"{'padded M=16 form' if old else 'M=24 K=12 form  '}: {t:.3f} ms  {abytes / t / 1e6:.0f} GB/s  "
              f"{flops / t / 1e9:.1f} TFLOP/s | with trace operand {tt:.3f} ms | max rel dev vs first {dev:.2e}", flush=True)


if __name__ == "__main__":
    main()
