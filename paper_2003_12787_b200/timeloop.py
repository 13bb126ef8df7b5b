"""The GPU time loop over several GPUs ("across GPUs this is one NVLink peer
copy ... of n^2 m doubles per boundary face").

One process per GPU (torchrun).  The periodic e^3 mesh is cut into z-slabs (shard.slab_partition);
each rank keeps its slab's state, material and predictor face buffers in HBM.  The face buffers
and the material are allocated with aderstp_device_alloc and exported once with CUDA IPC handles
(exchanged with all_gather_object), so every rank holds peer pointers to the two neighbouring
slabs' buffers.  aderstp_run_simulation_slab then runs the whole loop; its corrector kernel reads
the neighbours' boundary faces directly through those peer pointers (NVLink loads inside the
kernel that applies them: there is no separate halo copy and no halo buffer), and the ranks meet
twice per step in a host-side all_reduce of their stability flags (predictor done / corrector
done).  No kernel ever waits on another rank.

Multi-GPU execution needs several GPUs; the partition and synchronisation logic is covered by
the gloo tests (tests/test_multirank.py) and the slab kernels by the single-GPU multi-slab test
(tests/test_gpu_corrector.py), which drives the same C entry point with one slab per thread.
"""
from __future__ import annotations

from . import stp as _stp
from .shard import make_rank_sync, slab_neighbours, slab_partition


def run_simulation_distributed(plan, u_local, elements_per_dim: int, t_end: float, max_wavespeed: float,
                               par_local=None, cfl: float = 0.35, domain_len: float = 1.0, device=None):
    """Advance this rank's slab of the mesh to t_end (run_simulation, proj/src/solver.cpp:313-359).

    u_local: CUDA float64 tensor [e^2 nz, plan.q_size] (the slab's elements in global order);
    par_local: the slab's per-element material (elastic); max_wavespeed: the GLOBAL maximum (the
    same dt on every rank).  Returns (stable, steps, t_final)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    e = elements_per_dim
    z0, nz = slab_partition(e, world, rank)
    n_local = e * e * nz
    if u_local.shape[0] != n_local:
        raise ValueError("run_simulation_distributed: u_local does not hold this rank's slab")
    face_bytes = n_local * 6 * plan.face_size * 8
    own = {"face_q": _stp.device_alloc(face_bytes), "face_f": _stp.device_alloc(face_bytes)}
    if par_local is not None:  # the material goes to a shareable buffer too (per-face smax)
        own["par"] = _stp.device_alloc(n_local * 3 * 8)
        raw_view(own["par"], n_local * 3, par_local.device).copy_(par_local.reshape(-1))
        torch.cuda.synchronize()
    opened = []
    try:
        handles = {k: _stp.ipc_handle(v) for k, v in own.items()}
        everyone = [None] * world
        if world > 1:
            dist.all_gather_object(everyone, (z0, handles))
        else:
            everyone = [(z0, handles)]
        lo_rank, hi_rank = slab_neighbours(rank, world)

        def view(r):
            zb, hs = everyone[r]
            if r == rank:
                return own["face_q"], own["face_f"], own.get("par"), zb
            ptrs = {k: _stp.ipc_open(h) for k, h in hs.items()}
            opened.extend(ptrs.values())
            return ptrs["face_q"], ptrs["face_f"], ptrs.get("par"), zb

        lo = view(lo_rank)
        hi = lo if hi_rank == lo_rank else view(hi_rank)
        sync = make_rank_sync(device=device)
        par_dev = raw_view(own["par"], n_local * 3, u_local.device) if "par" in own else None
        return plan.run_simulation_slab(u_local, e, (z0, nz), own["face_q"], own["face_f"], t_end, max_wavespeed,
                                        lo=lo, hi=hi, par=par_dev, cfl=cfl, domain_len=domain_len, sync=sync)
    finally:
        for p in opened:
            _stp.ipc_close(p)
        if world > 1:
            dist.barrier()  # nobody reads this rank's buffers any more
        for p in own.values():
            _stp.device_free(p)


def raw_view(ptr: int, count: int, device):
    """A float64 tensor view of `count` doubles at a raw device pointer (no copy)."""
    import torch

    class _Raw:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False), "version": 2}

    return torch.as_tensor(_Raw(), device=device)
