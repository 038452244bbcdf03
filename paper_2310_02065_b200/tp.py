"""Tensor-parallel splits of the SpMM with the optional all-gather of C (SURVEY §8(e), §8(f)
rank 3; BASELINE.json north_star: "NCCL over NVLink is used only for the optional tensor-parallel
all-gather of C"). DESIGN.md §8.

Two splits:
- T-split (the data-parallel one bench.py scales): every rank holds the whole compressed A and a
  column slice of B; its slice of C is written token-major (below).
- Row split (V-block aligned, the weight-sharded one: each rank holds and compresses only its
  rows of A, e.g. a column-parallel linear layer): rank r computes C[rows_r, :] for all tokens;
  in row-major C those rows are one contiguous block, so the all-gather needs no re-layout
  either (``spmm_tp_rows_allgather``, fused: ``spmm_tp_rows_fused_allgather``).

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


# ------------------------------------------------------------------ row split (V-block aligned)
def row_slice(R: int, V: int, world: int, rank: int) -> Tuple[int, int]:
    """[r0, r1) of rank `rank` in an even split of the rows into whole V-blocks (a V-block's rows
    share column_idx, so a block cannot straddle ranks); requires R % (world·V) == 0 so every
    slice has equal size (all_gather_into_tensor needs equal shards)."""
    if V <= 0 or R % (world * V) != 0:
        raise ValueError(f"R={R} must be a multiple of world·V = {world * V}")
    per = R // world
    return rank * per, (rank + 1) * per


def shard_rows(x, r0: int, r1: int):
    """The compressed operand of rows [r0, r1) (whole V-blocks) as views of x's arrays: values and
    metadata rows, column_idx row blocks. (A rank that holds only its weight shard compresses its
    rows directly instead; both give the same arrays.)"""
    from . import VNMTensor
    if r0 % x.V or r1 % x.V:
        raise ValueError("row slices must be whole V-blocks")
    return VNMTensor(x.values[r0:r1], x.metadata[r0:r1], x.column_idx[r0 // x.V:r1 // x.V],
                     r1 - r0, x.K, x.V, x.M, x.N)


def gather_rows(c_local: torch.Tensor, out: Optional[torch.Tensor] = None, group=None) -> torch.Tensor:
    """All-gather the ranks' row blocks [R/world, T] of row-major C into C [R, T] (rank order = row
    order): contiguous blocks, one all_gather_into_tensor."""
    world = dist.get_world_size(group)
    Rl, T = c_local.shape
    if out is None:
        out = torch.empty((Rl * world, T), dtype=c_local.dtype, device=c_local.device)
    dist.all_gather_into_tensor(out, c_local.contiguous(), group=group)
    return out


def spmm_tp_rows_allgather(x_rows, B: torch.Tensor, bias_rows: Optional[torch.Tensor] = None,
                           out: Optional[torch.Tensor] = None, group=None, **kw) -> torch.Tensor:
    """C = A_vnm · B for all R rows on every rank from the row split: this rank's rows through
    venom_spmm (row-major C, its bias rows), then the NCCL all-gather. x_rows: this rank's
    compressed rows (shard_rows, or its own compressed weight shard); B: the full [K, T]."""
    from . import spmm
    c_local = spmm(x_rows, B, bias=bias_rows, **kw)
    return gather_rows(c_local, out=out, group=group)


def fused_rows_buffer(R: int, T: int, dtype, device, group=None):
    """The full row-major C [R, T] on every rank in symmetric memory, and its rendezvous handle."""
    import torch.distributed._symmetric_memory as symm_mem
    buf = symm_mem.empty((R, T), dtype=dtype, device=device)
    hdl = symm_mem.rendezvous(buf, group if group is not None else dist.group.WORLD)
    return buf, hdl


def peer_row_slices(hdl, r0: int, T: int, elem_size: int, rank: int):
    """Addresses where this rank's rows [r0, ...) start in every OTHER rank's full row-major C."""
    return [int(p) + r0 * T * elem_size for r, p in enumerate(hdl.buffer_ptrs) if r != rank]


def spmm_tp_rows_fused_allgather(x_rows, B: torch.Tensor, buf: torch.Tensor, hdl, bias_rows=None,
                                 group=None, **kw):
    """The row split with the all-gather fused into the SpMM epilogue: this rank's row block of C
    goes through the TMA-store epilogue into its own full buffer and, from the same staging slots,
    into every peer's buffer (opts.c_peers); a barrier on the symmetric-memory handle then orders
    every rank's stores before the buffer is read."""
    from . import spmm
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    R, T = buf.shape
    r0, r1 = row_slice(R, x_rows.V, world, rank)
    assert x_rows.R == r1 - r0
    spmm(x_rows, B, bias=bias_rows, out=buf[r0:r1],
         c_peers=peer_row_slices(hdl, r0, T, buf.element_size(), rank), **kw)
    hdl.barrier(channel=0)
    return buf
