"""Slice-sharded subspace extraction over ranks (NEXT-4).

Parallel-beam slices decouple (row p = (v N_r + r) N_c + c), and Eq. 4's
Lee-Seung iteration is row-local in its V half-step, so each rank holds the rows of a slice
range [r0, r1) -- every view of its slices -- and runs the V half-step on them; the D half-step
needs only the column sums B = V^T Y+ (K x N_k), H = V^T V (K x K) and two scalars, which one
all-reduce per iteration combines.  Every rank then applies the identical D update.  FBP and
synthesis are slice-local (no communication).

Host orchestration only: every arithmetic step runs in libhsnct's kernels (hsnct_nmf_begin /
_rowpass / _dupdate); the collective is the caller's process group (NCCL over NVLink on GPUs,
gloo in the CPU tests).
"""
from __future__ import annotations

import torch


def slice_range(Nr: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous slice range [r0, r1) of `rank` (the first Nr % world ranks get one more)."""
    base, extra = divmod(Nr, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def slice_rows(Nv: int, Nr: int, Nc: int, r0: int, r1: int) -> torch.Tensor:
    """Global row indices p = (v N_r + r) N_c + c of the slices [r0, r1), in the local row order
    (v, r - r0, c) of a rank whose handle has geometry (N_v, r1 - r0, N_c)."""
    v = torch.arange(Nv).view(Nv, 1, 1)
    r = torch.arange(r0, r1).view(1, r1 - r0, 1)
    c = torch.arange(Nc).view(1, 1, Nc)
    return ((v * Nr + r) * Nc + c).reshape(-1)


def default_allreduce(group=None):
    """Sum `red` over the ranks of `group` in place (torch.distributed; CUDA tensors go through a
    host copy on backends without CUDA support, e.g. gloo)."""
    import torch.distributed as dist

    def f(red: torch.Tensor):
        if not dist.is_initialized() or dist.get_world_size(group) == 1:
            return
        if red.is_cuda and dist.get_backend(group) != "nccl":
            host = red.cpu()
            dist.all_reduce(host, group=group)
            red.copy_(host)
        else:
            dist.all_reduce(red, group=group)
    return f


def sharded_subspace_decompose(h, Y, V, D, n_iter: int, obj_trace=None, allreduce=None, ws=None, red=None):
    """Eq. 4 (n_iter Lee-Seung iterations) on the union of the ranks' rows.  h: this rank's handle
    (local geometry); Y, V: this rank's rows; D: the full basis (identical on every rank, updated
    in place on every rank).  obj_trace (device fp64 [2 n_iter], nullable): the global objective
    after each half-step.  allreduce(red): in-place sum over ranks (default: torch.distributed)."""
    allreduce = default_allreduce() if allreduce is None else allreduce
    if red is None:
        red = torch.empty(h.nmf_red_size(), dtype=torch.float64, device=h.device)
    h.nmf_begin(Y, D, ws=ws)
    for it in range(n_iter):
        h.nmf_rowpass(Y, V, D, it, red, ws=ws)
        allreduce(red)
        h.nmf_dupdate(D, red, it, obj2=None if obj_trace is None else obj_trace[2 * it:2 * it + 2], ws=ws)
    return V, D
