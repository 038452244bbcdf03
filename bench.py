#!/usr/bin/env python
"""bench.py — V:N:M SpMM effective TFLOP/s on B200 (BASELINE.json metric), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl venom|reference]
                    [--workload NAME] [--scaling strong|weak]

One STEP is one pass of the whole hot path over one batch of
synthetic input: for every layer of the workload, venom_compress (a1-a3, plus the execution form
the planner picks), venom_spmm (a5-a9) and venom_decompress (a4). The default workload is the
largest single-GPU configuration of BASELINE.json, configs[3]: the GPT-3-175B-shaped FFN layer
12288×49152 × 8192 tokens at 128:2:16 ("large layers", where the north star's ≥60 % target
applies). configs[1] (the BERT-large FFN pair at 64:2:8) is measured beside it as `secondary`.

value   = useful SpMM FLOPs of the step (2·nnz·T per layer, all ranks) / max-over-ranks device time
          (mean over K CUDA-graph replays of the step; median / p10 / p90 in `step_ms`)
e2e     = the same metric through the public API with the step's inputs copied host->device from
          pinned memory and the step's results copied back, inside the timed region
roofline: dominant kernel = venom_spmm; achieved = algorithmic FLOPs per launch / mean launch time
          (CUDA events on the launching stream), peak from MEASURED_PEAKS.json
cpu_baseline: the CPU oracle (oracle/) on a bounded sample of the same workload, rank 0, N = 1,
          single-thread and all-core, extrapolated to the full step and labelled so.
L2: a 512 MiB buffer is written before every timed step (outside the events).
Multi-GPU (torchrun): --scaling strong (default; configs[3] "column-sharded over 1/2/4/8 B200"):
the T = 8192 tokens of one global B are split into T/N column slices, every rank compresses the
replicated weight (deterministic, bit-identical), runs its slice of the SpMM and decompresses its
R/N row slice; no collective on the data path. The optional NCCL all-gather of C (tp.py) is timed
separately (`allgather_C`), never folded into `value`. --scaling weak: every rank runs the whole
workload on its own tokens.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "V:N:M SpMM effective TFLOP/s and speedup vs dense cuBLAS fp16 GEMM"
UNIT = "TFLOP/s"

WORKLOAD_SETS = {
    "bert_large_ffn_4096tok_64:2:8": ["bert_large_ffn2_1024x4096x4096_64:2:8",
                                      "bert_large_ffn1_4096x1024x4096_64:2:8"],
    "gpt3_ffn_12288x49152x8192_128:2:16": ["gpt3_ffn_12288x49152x8192_128:2:16"],
}
for _k in synth.WORKLOADS:
    WORKLOAD_SETS.setdefault(_k, [_k])
# BASELINE configs[3]: the largest configuration that fits one GPU (the headline at N = 1)
DEFAULT_WORKLOAD = "gpt3_ffn_12288x49152x8192_128:2:16"
SECONDARY_WORKLOAD = "bert_large_ffn_4096tok_64:2:8"  # BASELINE configs[1]

# Per-SM L2 -> SMEM landing ceiling (GB/s per SM) for the `feed` roofline, from the independent TMA
# microbenchmark (tools/microbench_feed.cu, profiles/r02_microbench_feed.txt): the best rate of
# contiguous tile boxes with 160 KB in flight per SM on all 148 SMs, no MMA (153 B/ns per SM;
# 110 B/ns with the sparse MMA reading the same shared memory; tile::gather4 rows reach 84 B/ns).
FEED_CEILING_GBPS_PER_SM = 153.0
# tile::gather4 rows (15 issuing warps, the sparse MMAs consuming the same stages): 81 B/ns per SM
# (profiles/r02_microbench_feed.txt) — the ceiling of the gathered (M > 4) operand's feed
GATHER4_CEILING_GBPS_PER_SM = 81.2
FEED_CEILING_SOURCE = ("tools/microbench_feed.cu: TMA tile boxes, 148 SMs, 160 KB in flight per SM, no MMA "
                       "(profiles/r02_microbench_feed.txt; gather4 rows: 84 B/ns per SM)")


def useful_flops(w, T=None) -> float:
    """2·nnz·T with nnz = R·K·2/M (values are R×K/M×2)."""
    return 2.0 * (w["R"] * (w["K"] // w["M"]) * 2) * (w["T"] if T is None else T)


def algorithmic_bytes(w, T=None) -> float:
    """values + metadata + column_idx + B + C (fp16)."""
    R, K, V, M = w["R"], w["K"], w["V"], w["M"]
    T = w["T"] if T is None else T
    nnz = R * (K // M) * 2
    return 2 * nnz + nnz / 4 + 4 * (R // V) * (K // M) + 2 * K * T + 2 * R * T


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), d.get("hbm_gbs", 6650.0), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


def step_stats(ms):
    """mean / median / p10 / p90 of per-step times (ms)."""
    a = np.asarray(ms, dtype=np.float64)
    return {"mean": round(float(a.mean()), 5), "median": round(float(np.median(a)), 5),
            "p10": round(float(np.percentile(a, 10)), 5), "p90": round(float(np.percentile(a, 90)), 5),
            "n": int(a.size)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


# ----------------------------------------------------------------------------- distributed
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(ws: int, backend: str):
    if ws > 1 and not torch.distributed.is_initialized():
        torch.distributed.init_process_group(backend=backend)


def max_over_ranks(x: float, ws: int, device=None) -> float:
    if ws <= 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        torch.distributed.barrier()


def aggregate(per_rank_units: float, ws: int, t_max_s: float) -> float:
    """Weak scaling: every rank processed `per_rank_units`; whole-job throughput over the max
    rank time."""
    return per_rank_units * ws / t_max_s


def shard(w, ws: int, rank: int, scaling: str):
    """This rank's share of a layer. strong: columns [t0, t1) of the one global B
    (T/ws each, a multiple of 8) and rows [r0, r1) of the decompression (whole V-blocks, the last
    rank takes the remainder); weak: the whole layer on the rank's own tokens."""
    R, T, V = w["R"], w["T"], w["V"]
    if scaling == "weak" or ws == 1:
        return 0, T, 0, R
    if T % (8 * ws) != 0:
        raise ValueError(f"strong scaling needs T={T} divisible by 8·{ws}")
    per = T // ws
    nrb = R // V
    rb_per = (nrb + ws - 1) // ws
    r0 = min(R, rank * rb_per * V)
    r1 = min(R, (rank + 1) * rb_per * V)
    return rank * per, (rank + 1) * per, r0, r1


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples the SM clock and clock-event (throttle) reasons through NVML from a background
    thread every ~2 ms while the timed region runs (the main thread mostly sleeps in CUDA syncs)."""
    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, index: int):
        import threading
        self.samples, self.reasons, self.smax = [], set(), None
        self.err = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as ex:  # pragma: no cover - no NVML on this host
            self.nv, self.err = None, repr(ex)
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        import time as _t
        while self.nv is not None and not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, const in self.REASONS:
                    if mask & getattr(self.nv, const, 0):
                        self.reasons.add(name)
            except Exception:
                pass
            _t.sleep(0.002)

    def stop(self):
        self._stop.set()
        self.t.join(timeout=2)
        if self.nv is None or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.smax, "reasons": [self.err or "no samples"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- GPU workload
class Layer:
    def __init__(self, name, device, rank, ws=1, scaling="strong", form="auto"):
        import paper_2310_02065_b200 as venom
        self.venom = venom
        self.name = name
        self.w = dict(synth.WORKLOADS[name])
        w = self.w
        sa, sb = synth.seeds(w["cfg"])
        self.t0, self.t1, self.r0, self.r1 = shard(w, ws, rank, scaling)
        self.T = self.t1 - self.t0
        self.A = synth.gaussian_device((w["R"], w["K"]), 0.02, synth.F16, sa, device)
        if scaling == "weak" and ws > 1:
            # per-rank tokens: rank r draws its own activations
            self.B = synth.gaussian_device((w["K"], w["T"]), 1.0, synth.F16, sb + 7919 * rank, device)
        else:
            # one global B (same seed on every rank); this rank's slice is a column view (ldb = T)
            Bg = synth.gaussian_device((w["K"], w["T"]), 1.0, synth.F16, sb, device)
            self.B = Bg[:, self.t0:self.t1]
        self.bias = synth.gaussian_device((w["R"],), 0.5, synth.F16, sb + 1, device)
        # execution form of the operand: the V:N:M arrays themselves, or the same matrix re-encoded
        # as V:2:4 (reading #18) when that runs faster on B200; either way with the
        # metadata in tensor-core order
        self.expand = (form == "2to4") or (form == "auto" and venom.prefers_2to4(w["R"], w["K"], self.T, w["V"], w["M"]))
        if self.expand:
            self.x, self.y = venom.compress_2to4(self.A, V=w["V"], M=w["M"], check=True)
        else:
            self.x = venom.compress(self.A, V=w["V"], M=w["M"], check=True)
            self.y = venom.order_metadata(self.x)
        self.C = torch.empty((w["R"], self.T), dtype=torch.float16, device=device)
        # this rank's decompression rows: a row slice of the compressed operand (whole V-blocks)
        V = w["V"]
        self.xd = venom.VNMTensor(self.x.values[self.r0:self.r1], self.x.metadata[self.r0:self.r1],
                                  self.x.column_idx[self.r0 // V:self.r1 // V], self.r1 - self.r0,
                                  w["K"], V, w["M"])
        self.D = torch.empty((self.r1 - self.r0, w["K"]), dtype=torch.float16, device=device)
        self.flops = useful_flops(w, self.T)
        self.launches = (1 if self.expand else 2) + 1 + (1 if self.r1 > self.r0 else 0)

    def compress(self, A=None):
        """a1-a3 (+ the execution form): one fused kernel for the V:2:4 form, else compress + the
        tensor-core ordering of the metadata (compress(out=x) refreshes x.metadata_tc)."""
        w = self.w
        A = self.A if A is None else A
        if self.expand:
            self.venom.compress_2to4(A, V=w["V"], M=w["M"], out=(self.x, self.y))
        else:
            self.venom.compress(A, V=w["V"], M=w["M"], out=self.x)

    def spmm(self, B=None, out=None, **kw):
        return self.venom.spmm(self.y, self.B if B is None else B, bias=self.bias,
                               out=self.C if out is None else out, **kw)  # a5-a9

    def decompress(self):
        if self.r1 > self.r0:
            self.venom.decompress(self.xd, out=self.D)  # a4


def make_step(layers, device, overlap: bool, full: bool, kw):
    """The step's kernels as a small DAG over three streams (overlap): layer l's compression only
    feeds layer l's SpMM and decompression, so later layers' compressions run beside the first
    SpMM and the decompressions (a4) beside the SpMMs."""
    side_c = torch.cuda.Stream(device)
    side_d = torch.cuda.Stream(device)
    comp_done = [torch.cuda.Event() for _ in layers]

    def step(spmm_events=None, part_events=None, serial=False):
        stream = torch.cuda.current_stream(device)  # the capture stream when recording a graph
        if not overlap or serial:
            if part_events is not None:
                part_events[0].record(stream)
            for L in layers:
                L.compress()
            if part_events is not None:
                part_events[1].record(stream)
            for i, L in enumerate(layers):
                if spmm_events is not None:
                    spmm_events[i][0].record(stream)
                L.spmm(**kw)
                if spmm_events is not None:
                    spmm_events[i][1].record(stream)
            if full:
                if part_events is not None:
                    part_events[2].record(stream)
                for L in layers:
                    L.decompress()
                if part_events is not None:
                    part_events[3].record(stream)
            return
        side_c.wait_stream(stream)
        side_d.wait_stream(stream)
        layers[0].compress()
        comp_done[0].record(stream)
        with torch.cuda.stream(side_c):
            for i, L in enumerate(layers[1:], 1):
                L.compress()
                comp_done[i].record(side_c)
        if full:
            with torch.cuda.stream(side_d):
                for i, L in enumerate(layers):
                    side_d.wait_event(comp_done[i])
                    L.decompress()
        for i, L in enumerate(layers):
            stream.wait_event(comp_done[i])
            L.spmm(**kw)
        stream.wait_stream(side_c)
        stream.wait_stream(side_d)
    return step


def ev_pair():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def run_gpu(args, ws, rank, local):
    import paper_2310_02065_b200 as venom
    # VENOM_BENCH_DEVICE / VENOM_BENCH_BACKEND: tools-only overrides that run several ranks on one
    # GPU over gloo (the multi-rank code path checked on a one-GPU box; timings meaningless)
    device = torch.device("cuda", int(os.environ.get("VENOM_BENCH_DEVICE", local)))
    torch.cuda.set_device(device)
    init_dist(ws, os.environ.get("VENOM_BENCH_BACKEND", "nccl"))
    layers = [Layer(n, device, rank, ws, args.scaling, args.form) for n in WORKLOAD_SETS[args.workload]]
    kw = {}
    if args.tile_t:
        kw["tile_t"] = args.tile_t
    if args.group_n:
        kw["group_n"] = args.group_n
    if args.strategy:
        kw["strategy"] = {"gather": 1, "densek": 2}[args.strategy]
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream(device)
    full = args.step == "full"
    step = make_step(layers, device, args.overlap, full, kw)
    launches_per_step = sum(L.launches if full else L.launches - (1 if L.r1 > L.r0 else 0) for L in layers)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize(device)
    graph = None
    if args.graph:
        # the whole step as one CUDA graph (all streams): no per-launch CPU/driver gaps
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize(device)
        for _ in range(3):
            flush.zero_()
            graph.replay()
        torch.cuda.synchronize(device)

    # serial eager pass: per-kernel events (roofline per launch, step breakdown); the kernels run
    # alone here, as ncu sees them
    sp_ev = [[ev_pair() for _ in layers] for _ in range(args.steps)]
    pt_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()
        step(sp_ev[k], pt_ev[k], serial=True)
    torch.cuda.synchronize(device)
    spmm_ms = [[a.elapsed_time(b) for a, b in row] for row in sp_ev]
    compress_ms = statistics.mean(r[0].elapsed_time(r[1]) for r in pt_ev)
    decompress_ms = statistics.mean(r[2].elapsed_time(r[3]) for r in pt_ev) if full else 0.0

    # timed pass: the step (captured graph, or eager) K times, L2 flushed before each, events on
    # the launching stream, NVML clocks sampled throughout
    clocks = ClockSampler(device.index if device.index is not None else 0)
    gev = [ev_pair() for _ in range(args.steps)]
    barrier(ws)
    torch.cuda.synchronize(device)
    for k in range(args.steps):
        flush.zero_()
        gev[k][0].record(stream)
        if graph is not None:
            graph.replay()
        else:
            step()
        gev[k][1].record(stream)
    torch.cuda.synchronize(device)
    barrier(ws)
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in gev]
    total_s = max_over_ranks(sum(step_ms) / 1e3, ws, device)
    flops_rank = sum(L.flops for L in layers)
    # strong: the ranks' equal T-slices add up to the global T; weak: every rank ran the whole layer
    flops_job = flops_rank * ws
    value = flops_job * args.steps / total_s / 1e12
    ms_per_step = total_s * 1e3 / args.steps

    # dominant kernel: venom_spmm (per launch, serial pass)
    per_launch_ms = [statistics.mean(spmm_ms[k][i] for k in range(args.steps)) for i in range(len(layers))]
    spmm_flops = [L.flops for L in layers]
    achieved = sum(spmm_flops) / (sum(per_launch_ms) / 1e3) / 1e12
    peak_burst, peak_sust, hbm, peak_src = load_peaks()
    traffic, feed = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof) and ws == 1:
        with open(prof) as f:
            tr = json.load(f).get(args.workload)
        if tr:
            traffic = tr.get("dram_bytes_per_launch")
            xb = tr.get("l2_to_smem_bytes_per_launch")
            if xb and len(xb) == len(per_launch_ms):
                # the on-chip feed: L2 -> SMEM bytes per launch (ncu
                # l1tex__m_xbar2l1tex_read_bytes) over the live launch time, against the
                # independently measured per-SM landing ceiling × SMs
                ach = sum(xb) / (sum(per_launch_ms) / 1e3) / 1e9
                ceil = FEED_CEILING_GBPS_PER_SM * torch.cuda.get_device_properties(device).multi_processor_count
                feed = {"l2_to_smem_bytes_per_launch": xb, "achieved_GBps": round(ach, 1),
                        "ceiling_GBps": round(ceil, 1), "frac": round(ach / ceil, 4),
                        "ceiling_source": FEED_CEILING_SOURCE, "traffic_source": tr.get("source")}
                if all(L.w["M"] > 4 and not L.expand for L in layers):
                    # the gathered operand lands through tile::gather4, whose independently
                    # measured per-SM rate (with the sparse MMAs consuming) is its own ceiling
                    gceil = GATHER4_CEILING_GBPS_PER_SM * torch.cuda.get_device_properties(device).multi_processor_count
                    feed["gather4_ceiling_GBps"] = round(gceil, 1)
                    feed["frac_of_gather4"] = round(ach / gceil, 4)
    roofline = {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak_burst, "unit": "TFLOP/s",
                "frac": round(achieved / peak_burst, 4), "traffic": traffic,
                "frac_of_nominal_2250": round(achieved / 2250.0, 4),
                "peak_source": f"{peak_src} bf16 dense burst (MEASURED_PEAKS.json; fp16 runs at the same rate); "
                               f"useful FLOPs of a 2:4 sparse MMA are half its issued FLOPs, so the "
                               f"useful-FLOP peak equals the dense peak",
                "algorithmic_flops_per_launch": [int(x) for x in spmm_flops],
                "mean_launch_ms": [round(x, 5) for x in per_launch_ms],
                "hbm_frac": round(sum(algorithmic_bytes(L.w, L.T) for L in layers) / (sum(per_launch_ms) / 1e3) / 1e9 / hbm, 4),
                "feed": feed}

    # cuBLAS dense fp16 baseline at the same shapes (speedup metric)
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    cub = []
    for L in layers:
        dense = venom.decompress(L.x)
        ts = []
        for k in range(max(5, args.steps // 4) + 2):
            flush.zero_()
            a, b = ev_pair()
            a.record(stream)
            torch.matmul(dense, L.B)
            b.record(stream)
            ts.append((a, b))
        torch.cuda.synchronize(device)
        cub.append(statistics.median(a.elapsed_time(b) for a, b in ts[2:]))
        del dense
    speedup = [c / s for c, s in zip(cub, per_launch_ms)]

    # the optional tensor-parallel all-gather of C (tp.py), timed separately (N > 1, strong): the
    # token-major SpMM followed by NCCL all_gather_into_tensor, and the fused variant whose epilogue
    # stores the slice into every rank's symmetric-memory buffer (opts.c_peers) + a barrier
    allgather = None
    if ws > 1 and args.scaling == "strong":
        from paper_2310_02065_b200 import tp
        L = layers[0]
        c_tm = venom.spmm(L.y, L.B, bias=L.bias, transposed_out=True)
        full_tm = torch.empty((L.T * ws, L.w["R"]), dtype=c_tm.dtype, device=device)

        def timed(fn, n=10):
            for _ in range(3):
                fn()
            torch.cuda.synchronize(device)
            barrier(ws)
            a, b = ev_pair()
            a.record(stream)
            for _ in range(n):
                fn()
            b.record(stream)
            torch.cuda.synchronize(device)
            return max_over_ranks(a.elapsed_time(b) / n, ws, device)

        allgather = {"bytes_received_per_rank": int(c_tm.numel() * 2 * (ws - 1)),
                     "what": "tensor-parallel all-gather of C (tp.py), not in value"}
        try:
            allgather["allgather_ms"] = round(timed(lambda: tp.gather_token_major(c_tm, out=full_tm)), 4)
            allgather["spmm_then_allgather_ms"] = round(
                timed(lambda: tp.spmm_tp_allgather(L.y, L.B, bias=L.bias, out=full_tm)), 4)
        except Exception as e:  # e.g. a backend without all_gather_into_tensor on CUDA tensors
            allgather["unfused"] = f"unavailable: {e!r}"[:200]
        try:
            buf, hdl = tp.fused_allgather_buffer(L.w["R"], L.T * ws, torch.float16, device)
            fused_ms = timed(lambda: tp.spmm_tp_fused_allgather(L.y, L.B, buf, hdl, bias=L.bias))
            ok = bool(torch.equal(buf, full_tm))
            allgather.update({"spmm_fused_allgather_ms": round(fused_ms, 4), "fused_equals_nccl": ok})
        except Exception as e:  # symmetric memory unavailable
            allgather["fused"] = f"unavailable: {e!r}"[:200]

    # e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        hA = [L.A.cpu().pin_memory() for L in layers]
        hB = [L.B.cpu().pin_memory() for L in layers]
        hC = [torch.empty_like(L.C, device="cpu").pin_memory() for L in layers]
        dA = [torch.empty_like(L.A) for L in layers]
        dB = [torch.empty_like(hB[i], device=device) for i, L in enumerate(layers)]

        def e2e_step():
            for i, L in enumerate(layers):
                dA[i].copy_(hA[i], non_blocking=True)
                dB[i].copy_(hB[i], non_blocking=True)
            for i, L in enumerate(layers):
                L.compress(dA[i])
            for i, L in enumerate(layers):
                L.spmm(B=dB[i], **kw)
            if full:
                for L in layers:
                    L.decompress()
            for i, L in enumerate(layers):
                hC[i].copy_(L.C, non_blocking=True)
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize(device)
        ne = max(3, min(args.steps, 10))
        barrier(ws)
        a, b = ev_pair()
        a.record(stream)
        for _ in range(ne):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize(device)
        barrier(ws)
        e2e_s = max_over_ranks(a.elapsed_time(b) / 1e3, ws, device)
        h2d = sum(x.numel() * x.element_size() for x in hA + hB)
        d2h = sum(x.numel() * x.element_size() for x in hC)
        e2e = {"value": round(flops_job * ne / e2e_s / 1e12, 3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": ne}

    secondary = None
    if rank == 0 and ws == 1 and not args.no_secondary and args.workload != SECONDARY_WORKLOAD:
        secondary = measure_secondary(SECONDARY_WORKLOAD, device, flush, args.form)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(layers, budget_s=args.cpu_budget)

    if rank == 0:
        w0 = layers[0].w
        comp_bytes = sum(2 * L.w["R"] * L.w["K"] for L in layers)  # serial pass: every layer's A read once
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f16",
            "data": "synthetic (seeded; A ~ N(0,0.02^2), B ~ N(0,1), fp16)",
            "config": {"workload": args.workload, "layers": [L.name for L in layers],
                       "V:N:M": f"{w0['V']}:2:{w0['M']}", "tokens_total": sum(L.w["T"] for L in layers[:1]),
                       "tokens_per_gpu": layers[0].T,
                       "step": ("compress(+execution form)+spmm" + ("+decompress" if full else "") + " per layer"),
                       "operand_form": ["V:2:4 re-encoding, fused into compress (venom_compress_2to4)" if L.expand
                                        else "V:N:M (+ venom_order_metadata)" for L in layers],
                       "l2": "flushed (512 MiB write) before every timed step",
                       "parallelism": (f"T-split x{ws} (strong: column slices of one global B)" if args.scaling == "strong"
                                       else f"weak x{ws} (per-rank tokens)")},
            "step_ms": step_stats(step_ms),
            "spmm_only": {"tflops": round(achieved, 3), "ms_per_launch": [round(x, 5) for x in per_launch_ms],
                          "ms_per_launch_stats": [step_stats([spmm_ms[k][i] for k in range(args.steps)])
                                                  for i in range(len(layers))]},
            "step_breakdown_ms": {"compress_all_layers": round(compress_ms, 5),
                                  "spmm_all_layers": round(sum(per_launch_ms), 5),
                                  "decompress_all_layers": round(decompress_ms, 5),
                                  "measured_in": "serial eager pass (one stream, kernels alone)",
                                  "timed_as": ("CUDA graph replay of the step" if graph is not None else "eager step")
                                              + (" (compress of layers 2.. and decompress on side streams)" if args.overlap else ""),
                                  "compress_GBps": round(comp_bytes / compress_ms / 1e6, 1),
                                  "decompress_GBps": round(sum(2 * (L.r1 - L.r0) * L.w["K"] for L in layers) / decompress_ms / 1e6, 1)
                                  if decompress_ms > 0 else None},
            "speedup_vs_cublas": [round(s, 3) for s in speedup],
            "cublas_ms": [round(c, 5) for c in cub],
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "secondary": secondary,
            "allgather_C": allgather,
            "gpu_launches": launches_per_step * args.steps, "clocks": clk,
        }
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


def measure_secondary(workload, device, flush, form="auto", reps=20):
    """configs[1] beside the headline: per-layer SpMM launch time (median over `reps`, L2 flushed)
    and cuBLAS at the same shapes."""
    import paper_2310_02065_b200 as venom
    stream = torch.cuda.current_stream(device)
    out = {"workload": workload, "layers": []}
    tot_f, tot_ms = 0.0, 0.0
    for n in WORKLOAD_SETS[workload]:
        L = Layer(n, device, 0, 1, "strong", form)
        dense = venom.decompress(L.x)
        sp, cb = [], []
        for k in range(reps + 3):
            for fn, acc in ((lambda: L.spmm(), sp), (lambda: torch.matmul(dense, L.B), cb)):
                flush.zero_()
                a, b = ev_pair()
                a.record(stream)
                fn()
                b.record(stream)
                if k >= 3:
                    acc.append((a, b))
        torch.cuda.synchronize(device)
        s = statistics.median(a.elapsed_time(b) for a, b in sp)
        c = statistics.median(a.elapsed_time(b) for a, b in cb)
        tot_f += L.flops
        tot_ms += s
        out["layers"].append({"name": n, "spmm_ms": round(s, 5), "cublas_ms": round(c, 5),
                              "speedup_vs_cublas": round(c / s, 3),
                              "spmm_tflops": round(L.flops / s / 1e9, 2),
                              "operand_form": "V:2:4 (#18)" if L.expand else "V:N:M"})
        del L, dense
    out["spmm_tflops"] = round(tot_f / tot_ms / 1e9, 2)
    return out


# ----------------------------------------------------------------------------- CPU oracle
def _host_bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def cpu_baseline(layers, budget_s: float = 20.0, kind: str = "oracle"):
    """Time the CPU oracle (as it stands, never tuned) on a bounded sample of the workload and
    extrapolate to one full step: compression of a row-block subset, the SpMM on a token-column
    subset (all host cores, and single-threaded on a smaller subset), decompression of the same
    rows. The sample is stated in the result."""
    hosts = []
    for L in layers:
        w = L.w
        rows = min(w["R"], max(w["V"], ((1024 + w["V"] - 1) // w["V"]) * w["V"]))
        hosts.append((w, L.T, _host_bits(L.A[:rows]), _host_bits(L.B[:, :64])))
    return time_oracle(hosts, budget_s, kind)


def time_oracle(hosts, budget_s: float, kind: str = "oracle", single_thread: bool = True):
    """hosts: (workload, T of the rank, A row subset bits, B column subset bits). Returns the
    extrapolated full-step throughput of the oracle (all cores) plus the single-thread figure."""
    import oracle
    oracle.set_num_threads(0)
    cores = oracle.num_threads()
    t_step_all, t_step_one, flops, parts_desc = 0.0, 0.0, 0.0, []
    for w, T, A_sub, B_sub in hosts:
        R, K, V, M = w["R"], w["K"], w["V"], w["M"]
        rows = A_sub.shape[0]
        t0 = time.perf_counter()
        vals, meta, cidx = oracle.compress(A_sub, oracle.F16, V=V, M=M)
        t_c = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.decompress(vals, meta, cidx, rows, K, oracle.F16, V, M)
        t_d = time.perf_counter() - t0
        # SpMM: the full R needs the full compression; the sample multiplies the compressed row
        # subset by a column subset and scales by (R / rows) · (T / cols)
        share = max(0.5, budget_s / max(1, len(hosts)) - t_c - t_d)
        cols = 8
        t0 = time.perf_counter()
        oracle.spmm(vals, meta, cidx, rows, K, oracle.F16, V, M, np.ascontiguousarray(B_sub[:, :cols]))
        t_cal = time.perf_counter() - t0
        cols_all = int(min(B_sub.shape[1], max(8, cols * 0.6 * share / max(t_cal, 1e-4))))
        cols_all -= cols_all % 8
        t0 = time.perf_counter()
        oracle.spmm(vals, meta, cidx, rows, K, oracle.F16, V, M, np.ascontiguousarray(B_sub[:, :cols_all]))
        t_sp = time.perf_counter() - t0
        scale_r = R / rows
        t_full_all = (t_c + t_d) * scale_r + t_sp * scale_r * (T / cols_all)
        t_step_all += t_full_all
        if single_thread:
            oracle.set_num_threads(1)
            cols_one = 8
            t0 = time.perf_counter()
            oracle.spmm(vals, meta, cidx, rows, K, oracle.F16, V, M, np.ascontiguousarray(B_sub[:, :cols_one]))
            t_sp1 = time.perf_counter() - t0
            oracle.set_num_threads(0)
            t_step_one += (t_c + t_d) * scale_r + t_sp1 * scale_r * (T / cols_one)
        flops += 2.0 * R * (K // M) * 2 * T
        parts_desc.append(f"{R}x{K}x{T}: compress+decompress of {rows}/{R} rows ({t_c + t_d:.2f}s), "
                          f"SpMM of those rows on {cols_all}/{T} token columns ({t_sp:.2f}s, {cores} threads)")
    out = {"value": flops / t_step_all / 1e12, "unit": UNIT, "cores": cores, "kind": kind,
           "cpu_model": cpu_model(),
           "sample": "extrapolated to the full step from: " + "; ".join(parts_desc),
           "extrapolated_step_s": round(t_step_all, 2)}
    if single_thread:
        out["single_thread"] = {"value": flops / t_step_one / 1e12, "cores": 1,
                                "extrapolated_step_s": round(t_step_one, 2),
                                "sample": "SpMM on 8 token columns single-threaded; compression as above"}
    return out


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only), on the same
    workload, each step a bounded sample extrapolated to the full step."""
    if rank != 0:
        return
    hosts = []
    for n in WORKLOAD_SETS[args.workload]:
        w = dict(synth.WORKLOADS[n])
        sa, sb = synth.seeds(w["cfg"])
        rows = min(w["R"], w["V"] * max(1, 256 // w["V"]))
        # the first rows of the same seeded A (row-major draws: a prefix of the full matrix)
        A = synth.gaussian((rows, w["K"]), 0.02, synth.F16, sa)
        B = synth.gaussian((w["K"], 64), 1.0, synth.F16, sb)
        hosts.append((w, w["T"], A, B))
    per_step = max(1.0, min(6.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(min(args.warmup, 3)):
        time_oracle(hosts, per_step, single_thread=False)
    vals, secs, last = [], [], None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        last = time_oracle(hosts, per_step, kind="oracle", single_thread=False)
        secs.append(time.perf_counter() - t0)
        vals.append(last["value"])
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": last["extrapolated_step_s"] * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; same recipe as the GPU arm)",
            "config": {"workload": args.workload, "layers": WORKLOAD_SETS[args.workload],
                       "step": "oracle compress + SpMM + decompress, sampled and extrapolated per step",
                       "sample_wall_s_per_step": round(statistics.mean(secs), 3)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "oracle",
                             "cpu_model": last["cpu_model"], "sample": last["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["venom", "reference"], default="venom")
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOAD_SETS))
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong")
    ap.add_argument("--step", choices=["full", "spmm"], default="full")
    ap.add_argument("--tile-t", type=int, default=0)
    ap.add_argument("--group-n", type=int, default=0, help="tile-order group width (0: the planner's)")
    ap.add_argument("--strategy", choices=["gather", "densek"], default=None,
                    help="force a venom_spmm strategy (default: the library's planner)")
    ap.add_argument("--form", choices=["auto", "vnm", "2to4"], default="auto",
                    help="SpMM operand form: V:N:M as compressed, or re-encoded V:2:4 (venom_expand_2to4)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time the eager step instead of its CUDA-graph replay")
    ap.add_argument("--no-overlap", dest="overlap", action="store_false",
                    help="run every kernel of the step on one stream")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args(argv)
    args.warmup = max(3, args.warmup)
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import paper_2310_02065_b200 as venom
    venom.lib()  # fail loudly if the CUDA library is missing
    run_gpu(args, ws, rank, local)


if __name__ == "__main__":
    main()
