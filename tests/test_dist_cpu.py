"""World-size-2 gloo tests of the multi-GPU host logic on CPU:
the library's row partitioner and halo planner (srk_partition_rows /
srk_plan_create, host code of libsrk.so) drive a numpy simulation of exactly the
data movement the GPU path performs — pack the planned send rows, exchange them
with point-to-point messages, multiply the local CSR (renumbered columns) by the
[owned; ghost] block, all-reduce the per-rank Gram partials — and the result
must equal the global product and Gram."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import scipy.sparse as sp
    import torch

    import synth
    import paper_1504_04395_b200 as srk
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if case == "stencil":
            A = synth.conv_diff_3d(9, dtype=np.complex128, shift=-0.1j)
            cplx = True
        else:
            A = synth.random_sparse(400, 5, seed=3)
            cplx = False
        As = A.to_scipy()
        s = 3
        P = synth.random_rhs(A.n, s, 7, cplx)
        Y = synth.random_rhs(A.n, s, 8, cplx)
        off = srk.partition_rows(A.row_ptr, world)
        results = {}
        for name, M in (("A", As), ("AH", As.conj().T.tocsr())):
            M.sort_indices()
            plan = srk.make_plan(M.indptr, M.indices, off, rank)
            o0, o1 = plan.off0, plan.off1
            nl, ng = plan.n_local, plan.ghosts.size
            assert nl == o1 - o0
            P_loc = P[o0:o1]
            # halo exchange per the plan (what comm_halo does with ncclSend/ncclRecv)
            ext = np.zeros((nl + ng, s), dtype=P.dtype)
            ext[:nl] = P_loc
            soff = np.concatenate([[0], np.cumsum(plan.send_counts)])
            roff = np.concatenate([[0], np.cumsum(plan.recv_counts)])
            reqs = []
            for p in range(world):
                if p == rank:
                    continue
                if plan.send_counts[p]:
                    buf = torch.from_numpy(np.ascontiguousarray(P_loc[plan.send_local[soff[p]:soff[p + 1]]]).view(np.float64))
                    reqs.append(dist.isend(buf, dst=p))
            for p in range(world):
                if p == rank or not plan.recv_counts[p]:
                    continue
                rb = torch.zeros((plan.recv_counts[p], s * (2 if cplx else 1)), dtype=torch.float64)
                dist.recv(rb, src=p)
                ext[nl + roff[p]: nl + roff[p + 1]] = rb.numpy().view(P.dtype).reshape(-1, s)
            for r in reqs:
                r.wait()
            # ghost rows received must be exactly the planned global rows
            assert np.array_equal(ext[nl:], P[plan.ghosts])
            lo, hi = M.indptr[o0], M.indptr[o1]
            Mloc = sp.csr_matrix((M.data[lo:hi], plan.col, plan.row_ptr), shape=(nl, nl + ng))
            Q_loc = Mloc @ ext
            # fused Gram partial + all-reduce (what the finalize + ncclAllReduce do)
            g = torch.from_numpy(np.ascontiguousarray((Y[o0:o1].conj().T @ Q_loc)).view(np.float64).copy())
            dist.all_reduce(g)
            results[name] = (o0, o1, Q_loc, g.numpy().view(P.dtype).reshape(s, s))
        out_q.put((rank, results, P, Y, off))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["stencil", "random"])
def test_two_rank_halo_spmm_and_gram(case):
    import scipy.sparse as sp  # noqa: F401

    import synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda t: t[0])
    P, Y, off = outs[0][2], outs[0][3], outs[0][4]
    if case == "stencil":
        A = synth.conv_diff_3d(9, dtype=np.complex128, shift=-0.1j)
    else:
        A = synth.random_sparse(400, 5, seed=3)
    As = A.to_scipy()
    assert off[0] == 0 and off[-1] == A.n and np.all(np.diff(off) > 0)
    for name, M in (("A", As), ("AH", As.conj().T.tocsr())):
        Q = M @ P
        Qd = np.vstack([o[1][name][2] for o in outs])
        # same entries in the same per-row order: bitwise equal to the global product
        assert np.array_equal(Qd, Q), name
        G = Y.conj().T @ Q
        for o in outs:
            assert np.allclose(o[1][name][3], G, rtol=1e-13, atol=1e-13 * np.abs(G).max())
        # every rank holds the same all-reduced Gram (deterministic reduction)
        assert np.array_equal(outs[0][1][name][3], outs[1][1][name][3])


def test_partition_balances_nnz():
    import synth
    import paper_1504_04395_b200 as srk
    A = synth.power_law(20000, seed=4)
    for world in (2, 4, 8):
        off = srk.partition_rows(A.row_ptr, world)
        nnz = np.diff(A.row_ptr[off])
        assert nnz.max() - nnz.min() <= 2 * 512 + 1  # within one max row of perfect balance
        # plans of all ranks are mutually consistent: what p sends to q is what q expects from p
        plans = [srk.make_plan(A.row_ptr, A.col_idx, off, r) for r in range(world)]
        for p in range(world):
            soff = np.concatenate([[0], np.cumsum(plans[p].send_counts)])
            for qq in range(world):
                sent = plans[p].send_local[soff[qq]:soff[qq + 1]] + plans[p].off0
                roff = np.concatenate([[0], np.cumsum(plans[qq].recv_counts)])
                expected = plans[qq].ghosts[roff[p]:roff[p + 1]]
                assert np.array_equal(sent, expected)


@pytest.mark.parametrize("cplx", [False, True])
def test_csr_adjoint_host_matches_conj_transpose(cplx):
    """srk_csr_adjoint_host (a0 of the distributed operator) equals the
    textbook conj(A)^T entry for entry, columns ascending within each row."""
    import sys
    sys.path.insert(0, ROOT)
    import paper_1504_04395_b200 as srk
    import synth
    A = synth.random_sparse(500, 6, seed=11, dtype=np.complex128 if cplx else np.float64)
    As = A.to_scipy()
    rp, ci, va = srk.csr_adjoint_host(A.row_ptr, A.col_idx, A.values)
    T = As.conj().T.tocsr()
    T.sort_indices()
    assert np.array_equal(rp, T.indptr) and np.array_equal(ci, T.indices)
    assert np.array_equal(va, T.data)
    for i in range(A.n):
        assert np.all(np.diff(ci[rp[i]:rp[i + 1]]) > 0)
