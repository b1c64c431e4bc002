"""Element-slab domain decomposition of the exponential-DG hot path.

Host-side plumbing of the multi-GPU path: which elements a rank owns, which
face-trace layers it sends to / receives from its two slab neighbours before
every operator application, and the global reductions of the Gram-Schmidt
sweeps (one allreduce of k+1 doubles per sweep; the p augmentation scalars of
the phi vector live on rank 0 only and are added to rank 0's partials).

Slabs are cut along the slowest element axis (y for 2D meshes, z for 3D), so a
rank's elements and DOFs are one contiguous range of the reference's
element-major FieldState layout (proj/include/expdg/mesh.hpp:61-80) and the
halo is one element layer per side.  The tensors exchanged are whole element
layers (the LDG Burgers operator needs the neighbour's full elements for its
gradient; Euler only reads the face traces, which are a subset).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple


def slab_ranges(n: int, parts: int) -> List[Tuple[int, int]]:
    """Balanced contiguous ranges [start, stop) of n element layers over parts ranks."""
    if parts < 1 or n < parts:
        raise ValueError("need at least one element layer per rank")
    base, extra = divmod(n, parts)
    out, s = [], 0
    for r in range(parts):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


@dataclass
class SlabPlan:
    kind: str          # burgers1d | burgers2d | euler2d | euler3d
    order: int
    nx: int
    ny: int
    nz: int
    parts: int
    rank: int

    def __post_init__(self):
        dims = {"burgers1d": 1, "burgers2d": 2, "euler2d": 2, "euler3d": 3}[self.kind]
        self.dims = dims
        self.comps = {"burgers1d": 1, "burgers2d": 1, "euler2d": 4, "euler3d": 5}[self.kind]
        self.npe = (self.order + 1) ** dims
        self.layers = {1: self.nx, 2: self.ny, 3: self.nz}[dims]
        self.layer_elems = {1: 1, 2: self.nx, 3: self.nx * self.ny}[dims]
        self.start, self.stop = slab_ranges(self.layers, self.parts)[self.rank]

    # ---- ownership
    @property
    def block(self) -> int:
        """doubles per element"""
        return self.npe * self.comps

    @property
    def local_layers(self) -> int:
        return self.stop - self.start

    @property
    def local_dofs(self) -> int:
        return self.local_layers * self.layer_elems * self.block

    @property
    def dof_offset(self) -> int:
        return self.start * self.layer_elems * self.block

    @property
    def tail_here(self) -> bool:
        """the p augmentation scalars of the phi vector live on rank 0"""
        return self.rank == 0

    # ---- halo (periodic neighbours along the slab axis)
    @property
    def down(self) -> int:
        return (self.rank - 1) % self.parts

    @property
    def up(self) -> int:
        return (self.rank + 1) % self.parts

    def layer_range(self, layer: int) -> Tuple[int, int]:
        """global DOF range of one element layer"""
        layer %= self.layers
        s = layer * self.layer_elems * self.block
        return s, s + self.layer_elems * self.block

    def send_down(self) -> Tuple[int, int]:
        """my first layer, in local DOF coordinates (the down neighbour's upper halo)"""
        return 0, self.layer_elems * self.block

    def send_up(self) -> Tuple[int, int]:
        """my last layer, local coordinates (the up neighbour's lower halo)"""
        n = self.local_dofs
        return n - self.layer_elems * self.block, n

    def halo_layers(self) -> Tuple[int, int]:
        """global layer indices of the lower and upper halo"""
        return (self.start - 1) % self.layers, self.stop % self.layers


def exchange_halos(plan: SlabPlan, local, group=None):
    """Returns (lower_halo, upper_halo) element layers of `local` (a 1-D torch
    tensor of the rank's DOFs) from the neighbours.  Periodic; with one rank the
    halos are the rank's own last / first layer."""
    import torch
    import torch.distributed as dist

    a, b = plan.send_down()
    c, d = plan.send_up()
    if plan.parts == 1:
        return local[c:d].clone(), local[a:b].clone()
    lower = torch.empty(b - a, dtype=local.dtype, device=local.device)
    upper = torch.empty(d - c, dtype=local.dtype, device=local.device)
    # tags keep the two directions apart when down == up (two ranks)
    ops = [dist.P2POp(dist.isend, local[a:b].contiguous(), plan.down, group, tag=1),
           dist.P2POp(dist.isend, local[c:d].contiguous(), plan.up, group, tag=2),
           dist.P2POp(dist.irecv, lower, plan.down, group, tag=2),
           dist.P2POp(dist.irecv, upper, plan.up, group, tag=1)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    return lower, upper


def allreduce_partials(partials, group=None):
    """Sum of per-rank partial dots / norms (in place): one collective per sweep."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group)
    return partials
