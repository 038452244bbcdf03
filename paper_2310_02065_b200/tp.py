"""Tensor-parallel T-split of the SpMM with the optional all-gather of C (
BASELINE.json north_star: "NCCL over NVLink is used only for the optional tensor-parallel
all-gather of C"). DESIGN.md §8.

Each rank owns a contiguous slice of the T (token) columns of B and computes its slice of C with no
collective. To assemble the full output every rank holds, the slices are all-gathered. Each rank
writes its slice token-major (``spmm(..., transposed_out=True)``, C^T rows = tokens), so the slices
are contiguous blocks of the full C^T and the gather is one ``all_gather_into_tensor`` with no
re-layout. The SpMM runs in the library's kernels; this module only plans the split and calls
torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist


def t_slice(T: int, world: int, rank: int, align: int = 8) -> Tuple[int, int]:
    """[t0, t1) of rank `rank` in an even T-split whose slices are multiples of `align` columns (the
    SpMM's T % 8 == 0 requirement); requires T % (world·align) == 0 so every slice has equal size
    (all_gather_into_tensor needs equal shards)."""
    if T % (world * align) != 0:
        raise ValueError(f"T={T} must be a multiple of world·align = {world * align}")
    per = T // world
    return rank * per, (rank + 1) * per


def gather_token_major(c_local_tm: torch.Tensor, out: Optional[torch.Tensor] = None,
                       group=None) -> torch.Tensor:
    """All-gather the ranks' token-major slices [T/world, R] into the full C^T [T, R] (rank order =
    token order)."""
    world = dist.get_world_size(group)
    Tl, R = c_local_tm.shape
    if out is None:
        out = torch.empty((Tl * world, R), dtype=c_local_tm.dtype, device=c_local_tm.device)
    dist.all_gather_into_tensor(out, c_local_tm.contiguous(), group=group)
    return out


def spmm_tp_allgather(x, B_local: torch.Tensor, bias: Optional[torch.Tensor] = None,
                      out: Optional[torch.Tensor] = None, group=None, **kw) -> torch.Tensor:
    """C^T = (A_vnm · B)^T for the full T on every rank: the local T-slice through venom_spmm
    (token-major output), then the NCCL all-gather. B_local: this rank's [K, T/world] slice (any
    row stride, e.g. a column view of the global B)."""
    from . import spmm
    c_local = spmm(x, B_local, bias=bias, transposed_out=True, **kw)
    return gather_token_major(c_local, out=out, group=group)


# ------------------------------------------------------------------ fused all-gather (§8(f) rank 3)
def fused_allgather_buffer(R: int, T: int, dtype, device, group=None):
    """The full token-major output C^T [T, R] on every rank, in symmetric memory (peer-mapped over
    NVLink / NVSwitch), and its rendezvous handle (the peers' buffer addresses and a barrier)."""
    import torch.distributed._symmetric_memory as symm_mem
    buf = symm_mem.empty((T, R), dtype=dtype, device=device)
    hdl = symm_mem.rendezvous(buf, group if group is not None else dist.group.WORLD)
    return buf, hdl


def peer_slices(hdl, t0: int, R: int, elem_size: int, rank: int):
    """Addresses where this rank's token rows [t0, ...) start in every OTHER rank's full buffer."""
    return [int(p) + t0 * R * elem_size for r, p in enumerate(hdl.buffer_ptrs) if r != rank]


def spmm_tp_fused_allgather(x, B_local: torch.Tensor, buf: torch.Tensor, hdl, bias=None, group=None, **kw):
    """The T-split SpMM with the all-gather fused into its epilogue: this rank's slice of C^T is
    stored into its own full buffer AND, by the same kernel, into every peer's buffer (peer-to-peer
    stores over NVLink, no separate collective; include/venom.h opts.c_peers). A barrier on the
    symmetric-memory handle then orders every rank's stores before the buffer is read.
    B_local: this rank's [K, T/world] column slice of the global B."""
    from . import spmm
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    T, R = buf.shape
    t0, t1 = t_slice(T, world, rank)
    assert B_local.shape[1] == t1 - t0
    spmm(x, B_local, bias=bias, out=buf[t0:t1], transposed_out=True,
         c_peers=peer_slices(hdl, t0, R, buf.element_size(), rank), **kw)
    hdl.barrier(channel=0)
    return buf
