"""World-size-N gloo worker for tests/test_dist_gloo.py (CPU only).

Emulates the multi-GPU data path of libqswg on the host: every rank takes
its row block from the library's partition planner (qswg_plan_rows), its
halo plan from qswg_plan_halo, exchanges exactly those hulls with gloo
send/recv (as comm_nccl.cpp does with ncclSend/ncclRecv), computes its rows
of y = L x with entries outside its own segment and received halos poisoned
with NaN, and reduces the stop-test maxima with allreduce(MAX).  Rank 0
checks the gathered result against the single-process SpMV of the C oracle.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_2003_02450_b200 import api, graphs  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    port = Oracle("port")
    failures = 0
    for name, size in (("c2", 6), ("c5", 4), ("c3", 40), ("c1", 24)):
        w = graphs.config(name, size=size)
        n, dim = w.n, w.dim
        L = port.build(w).csr()
        colptr = L.indptr[np.arange(n + 1) * n]
        starts = api.plan_rows(n, colptr, world)
        # partition: monotone, on rho-column boundaries, covering [0, dim)
        assert starts[0] == 0 and starts[-1] == dim and np.all(np.diff(starts) >= 0)
        assert np.all(starts % n == 0)
        r0, r1 = int(starts[rank]), int(starts[rank + 1])
        cols = L.indices[L.indptr[r0]:L.indptr[r1]]
        lo, hi = api.plan_halo(cols, starts, rank)
        table_lo = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        table_hi = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(table_lo, torch.from_numpy(lo))
        dist.all_gather(table_hi, torch.from_numpy(hi))
        rng = np.random.default_rng(5)
        x_true = rng.uniform(-1, 1, dim) + 1j * rng.uniform(-1, 1, dim)
        x = np.full(dim, np.nan + 1j * np.nan)
        x[r0:r1] = x_true[r0:r1]
        # halo exchange: send what each peer needs from me, receive my needs
        reqs = []
        xr = torch.from_numpy(x.view(np.float64))
        for q in range(world):
            if q == rank:
                continue
            slo, shi = int(table_lo[q][rank]), int(table_hi[q][rank])
            if shi > slo:
                reqs.append(dist.isend(xr[2 * slo:2 * shi].clone(), q))
            rlo, rhi = int(table_lo[rank][q]), int(table_hi[rank][q])
            if rhi > rlo:
                buf = torch.zeros(2 * (rhi - rlo), dtype=torch.float64)
                dist.recv(buf, q)
                x[rlo:rhi] = buf.numpy().view(np.complex128)
        for r in reqs:
            r.wait()
        # local rows of y = L x; any entry touching a non-received column is NaN
        y = np.zeros(r1 - r0, np.complex128)
        for r in range(r0, r1):
            b, e = L.indptr[r], L.indptr[r + 1]
            y[r - r0] = np.dot(L.data[b:e], x[L.indices[b:e]])
        # stop-test maxima: allreduce(MAX) of the bit patterns (non-negative doubles)
        m = torch.tensor([np.abs(y).max(initial=0.0)], dtype=torch.float64)
        bits = m.view(torch.int64).clone()
        dist.all_reduce(bits, op=dist.ReduceOp.MAX)
        gathered = [None] * world
        dist.all_gather_object(gathered, (r0, y))
        if rank == 0:
            y_full = np.zeros(dim, np.complex128)
            for g0, yy in gathered:
                y_full[g0:g0 + len(yy)] = yy
            want = port.build(w).spmv(x_true)
            finite = bool(np.isfinite(y_full).all())
            err = float(np.abs(y_full - want).max()) if finite else float("nan")
            # the allreduced max equals the max of the gathered rows exactly
            ok = finite and err <= 1e-13 * max(1, np.abs(want).max())
            ok = ok and bits.view(torch.float64).item() == np.abs(y_full).max()
            rows = np.diff(starts)
            print(f"{name}: world={world} starts={starts.tolist()} rows={rows.tolist()} finite={finite} err={err:.1e} ok={ok}", flush=True)
            failures += 0 if ok else 1
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
