"""Multi-process (gloo, CPU) tests of the latitude-band decomposition's host logic.

The CUDA library exchanges halo rows with NCCL (first local row -> rank-1, last -> rank+1) and
all-gathers fixed row-group partial sums.  These tests run that same exchange pattern with
torch.distributed/gloo over the binding's own partition (`band_rows`), apply the CPU oracle on each
rank's band plus ghost rows, and check that (a) every rank's rows equal the single-process oracle
apply bitwise and (b) the grouped global sums are bitwise identical for any rank count.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
import paper_1811_03852_b200 as egs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROB = gen.Problem(24, 16, 5, seed=6)   # 16 rows -> 8 groups of 2 rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _group_sums(rows_sum, ny, j0, j1):
    """sum of per-row partials inside each fixed row-group fully contained in [j0, j1)."""
    G = min(8, ny)
    out = []
    for g in range(G):
        a, b = g * ny // G, (g + 1) * ny // G
        if a >= j0 and b <= j1:
            s = 0.0
            for j in range(a, b):
                s += rows_sum[j - j0]
            out.append(s)
        else:
            assert b <= j0 or a >= j1, "a reduction group straddles two ranks"
    return out


def _worker(rank, ws, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        p = PROB
        nx, ny, nz = p.nx, p.ny, p.nz
        row = nx * nz
        j0, j1 = egs.band_rows(ny, rank, ws)
        # the global scaled operator and a global seeded field (every rank can make them)
        bands_all, _ = gen.host(p)
        ahat_all, _ = oracle.scale((nx, ny, nz), bands_all, "fp64")
        z_all = np.random.default_rng(123).standard_normal(p.n)
        z_loc = z_all[j0 * row:j1 * row].copy()
        # ---- halo exchange, the library's pattern (eg halo(): send first row to rank-1 and last
        # row to rank+1, receive the ghosts from them) ----
        lo = torch.zeros(row, dtype=torch.float64)
        hi = torch.zeros(row, dtype=torch.float64)
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(z_loc[:row].copy()), rank - 1))
            reqs.append(dist.irecv(lo, rank - 1))
        if rank < ws - 1:
            reqs.append(dist.isend(torch.from_numpy(z_loc[-row:].copy()), rank + 1))
            reqs.append(dist.irecv(hi, rank + 1))
        for r in reqs:
            r.wait()
        # ---- apply on band + ghost rows with the oracle ----
        e0 = j0 - 1 if j0 > 0 else j0
        e1 = j1 + 1 if j1 < ny else j1
        ext = [z_loc]
        if j0 > 0:
            ext.insert(0, lo.numpy())
        if j1 < ny:
            ext.append(hi.numpy())
        z_ext = np.concatenate(ext)
        a_ext = ahat_all[:, e0 * row:e1 * row].copy()
        # the sub-grid's artificial edges become "poles": zero the couplings across them
        if e0 != 0:
            a_ext[3, :row] = 0.0          # S band of the first ghost row
        if e1 != ny:
            a_ext[2, -row:] = 0.0         # N band of the last ghost row
        y_ext = oracle.apply((nx, e1 - e0, nz), a_ext, z_ext)
        y_loc = y_ext[(j0 - e0) * row:(j0 - e0) * row + (j1 - j0) * row]
        y_ref = oracle.apply((nx, ny, nz), ahat_all, z_all)[j0 * row:j1 * row]
        apply_ok = bool(np.array_equal(y_loc, y_ref))
        # ---- grouped global sum of z . y, all-gathered, groups summed in order ----
        rows_sum = [float(np.sum(z_loc[k * row:(k + 1) * row] * y_loc[k * row:(k + 1) * row]))
                    for k in range(j1 - j0)]
        mine = torch.tensor(_group_sums(rows_sum, ny, j0, j1), dtype=torch.float64)
        gathered = [torch.zeros_like(mine) for _ in range(ws)]
        dist.all_gather(gathered, mine)
        total = 0.0
        for t in torch.cat(gathered).tolist():
            total += t
        result_q.put((rank, apply_ok, total, (j0, j1)))
    finally:
        dist.destroy_process_group()


def _run(ws):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=120) for _ in range(ws)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return sorted(out)


def _serial_total():
    p = PROB
    row = p.nx * p.nz
    bands, _ = gen.host(p)
    ahat, _ = oracle.scale((p.nx, p.ny, p.nz), bands, "fp64")
    z = np.random.default_rng(123).standard_normal(p.n)
    y = oracle.apply((p.nx, p.ny, p.nz), ahat, z)
    rows_sum = [float(np.sum(z[j * row:(j + 1) * row] * y[j * row:(j + 1) * row])) for j in range(p.ny)]
    tot = 0.0
    for t in _group_sums(rows_sum, p.ny, 0, p.ny):
        tot += t
    return tot


@pytest.mark.parametrize("ws", [2, 4])
def test_band_decomposition_halo_and_grouped_sums_gloo(ws):
    out = _run(ws)
    serial = _serial_total()
    bands = [o[3] for o in out]
    assert bands[0][0] == 0 and bands[-1][1] == PROB.ny
    for rank, apply_ok, total, _ in out:
        assert apply_ok, f"rank {rank}: band apply with exchanged ghost rows differs from the global apply"
        assert total == serial, "grouped global sum is not bitwise invariant under the decomposition"
