"""Host-side logic of the slab-partitioned multi-GPU path,
exercised with world_size 2 over gloo on CPU: ownership, periodic halo layers,
and the per-sweep reductions of the distributed Gram-Schmidt (partials summed by
one allreduce; the augmentation tail counted once, on rank 0)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_01316_b200.partition import SlabPlan, allreduce_partials, exchange_halos, slab_ranges


def test_slab_ranges_cover_and_balance():
    for n, p in [(1024, 8), (7, 3), (64, 4), (5, 5)]:
        r = slab_ranges(n, p)
        assert r[0][0] == 0 and r[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        sizes = [b - a for a, b in r]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slab_ranges(3, 4)


def test_plan_layout_matches_fieldstate_order():
    plans = [SlabPlan("euler2d", 2, 8, 6, 1, 3, r) for r in range(3)]
    total = sum(p.local_dofs for p in plans)
    assert total == 8 * 6 * 9 * 4
    off = 0
    for p in plans:
        assert p.dof_offset == off
        off += p.local_dofs
    assert [p.tail_here for p in plans] == [True, False, False]
    p = SlabPlan("euler3d", 3, 4, 4, 8, 2, 1)
    assert p.layer_elems == 16 and p.halo_layers() == (3, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kind, order, nx, ny, nz = "euler2d", 2, 6, 8, 1
        plan = SlabPlan(kind, order, nx, ny, nz, world, rank)
        rng = np.random.default_rng(1234)
        n_glob = nx * ny * plan.block
        field = torch.tensor(rng.standard_normal(n_glob))
        a = plan.dof_offset
        local = field[a:a + plan.local_dofs].clone()
        lower, upper = exchange_halos(plan, local)
        lo, hi = plan.halo_layers()
        l0, l1 = plan.layer_range(lo)
        u0, u1 = plan.layer_range(hi)
        ok_halo = torch.equal(lower, field[l0:l1]) and torch.equal(upper, field[u0:u1])

        # distributed CGS2 sweep: k basis vectors + y of length n (+ p tail scalars on rank 0)
        k, p = 5, 1
        V = torch.tensor(rng.standard_normal((k, n_glob + p)))
        y = torch.tensor(rng.standard_normal(n_glob + p))
        sl = slice(a, a + plan.local_dofs)
        part = (V[:, sl] * y[sl]).sum(dim=1)
        if plan.tail_here:
            part += (V[:, n_glob:] * y[n_glob:]).sum(dim=1)
        dots = allreduce_partials(part.clone())
        ref = V @ y
        ok_dots = bool(torch.allclose(dots, ref, rtol=1e-12, atol=1e-12))
        # pass-B update on the local slab with the global coefficients, then the norm
        y_loc = y[sl] - V[:, sl].T @ dots
        nrm = (y_loc * y_loc).sum().reshape(1)
        if plan.tail_here:
            yt = y[n_glob:] - V[:, n_glob:].T @ dots
            nrm += (yt * yt).sum()
        nrm = allreduce_partials(nrm)
        y_ref = y - V.T @ ref
        ok_norm = abs(float(nrm) - float(y_ref @ y_ref)) <= 1e-10 * float(y_ref @ y_ref)
        flags = torch.tensor([int(ok_halo), int(ok_dots), int(ok_norm)])
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        if rank == 0:
            with open(result_path, "w") as f:
                f.write(" ".join(str(int(v)) for v in flags))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_halo_exchange_and_distributed_gram_schmidt(tmp_path, world):
    out = tmp_path / "flags.txt"
    mp.spawn(_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    assert out.read_text().split() == ["1", "1", "1"]
