"""World-size-2 tests of the multi-GPU host logic on CPU (gloo): bench.py's rank environment,
max-over-ranks timing, weak-scaling aggregation, rank-0-only reference arm, and the T-split of the
SpMM: column shards of B computed independently and concatenated equal the
unsharded product bit for bit (checked with the oracle, no GPU)."""
from __future__ import annotations

import io
import os
import socket
import sys
from contextlib import redirect_stdout

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, ws: int, port: int, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE=str(ws), LOCAL_RANK=str(rank))
        import bench
        import oracle
        import synth
        env = bench.dist_env()
        assert env == (ws, rank, rank), env
        bench.init_dist(ws, "gloo")
        # max over ranks and weak-scaling aggregation
        t = bench.max_over_ranks(0.5 + rank, ws)
        assert t == 0.5 + (ws - 1)
        assert bench.aggregate(10.0, ws, t) == pytest.approx(10.0 * ws / t)
        bench.barrier(ws)

        # strong scaling (bench.py --scaling strong, the default): bench.shard gives rank r the
        # columns [t0, t1) of the one global B and the rows [r0, r1) it decompresses; over the ranks
        # the column slices tile [0, T) and the row slices tile [0, R) in whole V-blocks
        w = dict(R=12288, K=49152, T=8192, V=128, M=16)
        sh = bench.shard(w, ws, rank, "strong")
        all_sh = [None] * ws
        dist.all_gather_object(all_sh, sh)
        assert [a[0] for a in all_sh] == [r * (8192 // ws) for r in range(ws)]
        assert all_sh[-1][1] == 8192 and all(all_sh[r][1] == all_sh[r + 1][0] for r in range(ws - 1))
        assert all_sh[0][2] == 0 and all_sh[-1][3] == 12288
        assert all(all_sh[r][3] == all_sh[r + 1][2] for r in range(ws - 1)) and all(a[2] % 128 == 0 for a in all_sh)
        assert bench.shard(w, ws, rank, "weak") == (0, 8192, 0, 12288)
        with pytest.raises(ValueError):
            bench.shard(dict(w, T=8 * ws + 4), ws, rank, "strong")
        # the job's useful FLOPs: strong-split ranks add up to the unsharded layer
        per_rank = bench.useful_flops(w, sh[1] - sh[0])
        tot = torch.tensor([per_rank], dtype=torch.float64)
        dist.all_reduce(tot)
        assert float(tot) == bench.useful_flops(w)

        # T-split: rank r owns columns [r*T/ws, (r+1)*T/ws) of one global B; no collective on the
        # SpMM itself, the all_gather below only collects the result for the check
        R, K, T, V, M = 64, 128, 96, 32, 8
        A = synth.gaussian((R, K), 0.02, synth.F16, 5)
        B = synth.gaussian((K, T), 1.0, synth.F16, 6)
        parts = oracle.compress(A, synth.F16, V=V, M=M)
        ts = T // ws
        C_r = oracle.spmm(*parts, R, K, synth.F16, V, M, np.ascontiguousarray(B[:, rank * ts:(rank + 1) * ts]))
        gathered = [torch.empty((R, ts), dtype=torch.float64) for _ in range(ws)]
        dist.all_gather(gathered, torch.from_numpy(C_r))
        if rank == 0:
            C_full = oracle.spmm(*parts, R, K, synth.F16, V, M, B)
            C_cat = torch.cat(gathered, dim=1).numpy()
            assert np.array_equal(C_cat, C_full)

        # tensor-parallel all-gather of C (paper_2310_02065_b200/tp.py): token-major slices gathered
        # with one all_gather_into_tensor equal the unsharded product transposed (the local products
        # stand in for the GPU SpMM with the oracle)
        from paper_2310_02065_b200 import tp
        t0, t1 = tp.t_slice(T, ws, rank)
        assert (t0, t1) == (rank * ts, (rank + 1) * ts)
        C_tm = torch.from_numpy(np.ascontiguousarray(C_r.T))          # [T/ws, R]
        full_tm = tp.gather_token_major(C_tm)
        if rank == 0:
            assert np.array_equal(full_tm.numpy(), oracle.spmm(*parts, R, K, synth.F16, V, M, B).T)
        with pytest.raises(ValueError):
            tp.t_slice(100, ws, rank)
        # fused all-gather addressing: this rank's slice [t0, t1) of C^T [T, R] lands at row t0 of
        # every OTHER rank's buffer (host arithmetic of tp.peer_slices)
        class _H:
            buffer_ptrs = [1 << 40, 2 << 40, 3 << 40][:ws]
        ps = tp.peer_slices(_H, t0, R, 2, rank)
        assert ps == [b + t0 * R * 2 for r, b in enumerate(_H.buffer_ptrs) if r != rank] and len(ps) == ws - 1

        # row split (tp.row_slice / shard_rows / gather_rows): rank r owns whole V-blocks of rows;
        # its oracle product on its compressed rows, gathered as row-major blocks, equals the
        # unsharded product bit for bit, and the row slices tile [0, R)
        r0, r1 = tp.row_slice(R, V, ws, rank)
        assert (r0, r1) == (rank * (R // ws), (rank + 1) * (R // ws)) and r0 % V == 0
        vals, meta, cidx = parts
        G = K // M
        part_r = (vals.reshape(R, G, 2)[r0:r1], meta[r0:r1], cidx.reshape(R // V, G, 4)[r0 // V:r1 // V])
        C_rows = oracle.spmm(*part_r, r1 - r0, K, synth.F16, V, M, B)
        full_rows = tp.gather_rows(torch.from_numpy(C_rows))
        if rank == 0:
            assert np.array_equal(full_rows.numpy(), oracle.spmm(*parts, R, K, synth.F16, V, M, B))
        # and the rank's own compression of its weight shard gives the same arrays (V-block aligned)
        own = oracle.compress(np.ascontiguousarray(A[r0:r1]), synth.F16, V=V, M=M)
        assert all(np.array_equal(a.reshape(-1), b.reshape(-1)) for a, b in zip(own, part_r))
        with pytest.raises(ValueError):
            tp.row_slice(R, 48, ws, rank)
        prs = tp.peer_row_slices(_H, r0, T, 2, rank)
        assert prs == [b + r0 * T * 2 for r, b in enumerate(_H.buffer_ptrs) if r != rank]

        # weak scaling draws per-rank activations: the ranks' B differ
        b_r = torch.from_numpy(synth.gaussian((8, 8), 1.0, synth.F16, 1001 + 7919 * rank).astype(np.int32))
        gb = [torch.empty_like(b_r) for _ in range(ws)]
        dist.all_gather(gb, b_r)
        assert not torch.equal(gb[0], gb[1])

        # --impl reference: rank 0 alone runs and prints; other ranks exit without work
        if rank != 0:
            out = io.StringIO()
            with redirect_stdout(out):
                bench.main(["--impl", "reference", "--gpus", str(ws), "--steps", "1", "--warmup", "3"])
            assert out.getvalue() == ""
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent instead of hanging it
        q.put((rank, repr(e)))


def test_two_rank_gloo_host_logic():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results
