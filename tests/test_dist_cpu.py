"""Multi-rank host logic of the row-sharded path, on CPU (gloo, world size 2 and 3).

Each rank takes its equal-nnz row block (mpsg_partition_rows, the reference's
kernels.hpp:63-80 rule), computes the column interval it reads, and runs the
library's halo plan (mpsg_halo_plan) against every rank's interval; the x halo
then moves rank to rank over gloo exactly as the NCCL send/recv group does on
the GPUs.  The local rows are multiplied by the C oracle against the assembled
global-length x -- with everything outside the planned interval poisoned to
NaN -- and the gathered y must equal the single-process reference SpMV bit for
bit in both exact orders.  This pins partition + plan + exchange; the device
kernels themselves are the single-GPU kernels (pinned by the gpu tests).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2412_17510_b200 as M
import synth

CASES = [  # (cfg, K, p1, p2, p3)
    (3, 2, 400, 8.0, 0.0),  # banded complex: neighbour halo
    (4, 2, 3000, 900.0, 1.8),  # power-law: all-to-all halo
    (5, 4, 10, 0.0, 0.0),  # 3D Laplacian: plane halo
    (2, 3, 800, 32.0, 0.0),  # random Poisson rows
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(xfull, send, recv, rank, P):
    import torch

    reqs, bufs = [], []
    for q in range(P):
        if q == rank:
            continue
        slo, shi = send[q]
        if shi > slo:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(xfull[slo:shi])), q))
        rlo, rhi = recv[q]
        if rhi > rlo:
            buf = torch.empty((rhi - rlo, xfull.shape[1]), dtype=torch.float64)
            bufs.append((rlo, rhi, buf))
            reqs.append(dist.irecv(buf, q))
    for r in reqs:
        r.wait()
    for rlo, rhi, buf in bufs:
        xfull[rlo:rhi] = buf.numpy()


def _worker(rank, P, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        out = []
        for cfg, K, p1, p2, p3 in CASES:
            A = synth.config_matrix(cfg, K, p1, p2, p3)
            cplx = cfg == 3
            xs = synth.config_vector(cfg, A.nrows, K)
            xs = list(xs) if cplx else [xs]
            bounds = M.partition_rows(A.indptr, A.nrows, P)
            b, e = int(bounds[rank]), int(bounds[rank + 1])
            loc = M.shard_rows(A, b, e)
            need = M.need_interval(loc, b, e)
            needs = [None] * P
            dist.all_gather_object(needs, need)
            send, recv = M.halo_plan(P, rank, bounds, np.array(needs).reshape(-1))
            plans = [None] * P
            dist.all_gather_object(plans, (send.tolist(), recv.tolist()))
            # what r sends to q is what q receives from r
            for r_ in range(P):
                for q_ in range(P):
                    assert plans[r_][0][q_] == plans[q_][1][r_], (r_, q_, plans)
            xfulls = []
            for x in xs:
                xf = np.full_like(x, np.nan)  # poison: only the planned interval may be read
                xf[b:e] = x[b:e]
                _exchange(xf, send, recv, rank, P)
                lo, hi = need
                assert not np.isnan(xf[lo:hi]).any()
                xfulls.append(xf)
            res = {}
            for order in (O.SCALAR, O.LANE4):
                if cplx:
                    yr, yi = O.spmv_complex(loc, xfulls[0], xfulls[1], order)
                    res[order] = (yr, yi)
                else:
                    res[order] = (O.spmv(loc, xfulls[0], order),)
            gathered = [None] * P
            dist.all_gather_object(gathered, res)
            if rank == 0:
                for order in (O.SCALAR, O.LANE4):
                    parts = [np.concatenate([g[order][j] for g in gathered]) for j in range(len(xs))]
                    if cplx:
                        ref = O.spmv_complex(A, xs[0], xs[1], order)
                    else:
                        ref = (O.spmv(A, xs[0], order),)
                    for p_, r_ in zip(parts, ref):
                        ok = p_.tobytes() == np.ascontiguousarray(r_).tobytes()
                        out.append((cfg, K, order, ok, int(sum(max(0, hi_ - lo_) for lo_, hi_ in recv))))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 3])
def test_row_sharded_spmv_bit_exact_over_gloo(P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, q)) for r in range(P)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out and all(ok for (_, _, _, ok, _) in out), out


def test_halo_plan_single_rank_is_empty():
    send, recv = M.halo_plan(1, 0, [0, 10], [0, 10])
    assert (send == 0).all() and (recv == 0).all()


def test_halo_plan_neighbour_band():
    # 3 ranks of 10 rows, bandwidth 2: each reads 2 rows from each neighbour
    bounds = [0, 10, 20, 30]
    need = [0, 12, 8, 22, 18, 30]
    send, recv = M.halo_plan(3, 1, bounds, need)
    assert send.tolist() == [[10, 12], [0, 0], [18, 20]]
    assert recv.tolist() == [[8, 10], [0, 0], [20, 22]]
