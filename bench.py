#!/usr/bin/env python
"""bench.py — V:N:M SpMM effective TFLOP/s on B200 (BASELINE.json metric), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl venom|reference] [--workload NAME]

One STEP is one pass of the whole hot path over one batch of
synthetic input: for every layer of the workload, venom_compress (a1-a3), venom_spmm (a5-a9) and
venom_decompress (a4). The default workload is BASELINE.json configs[1]: the two BERT-large FFN
linear layers (1024×4096 and 4096×1024) × 4096 tokens at 64:2:8.

value   = useful SpMM FLOPs (2·nnz·T per layer, all ranks) / max-over-ranks device time of K steps
e2e     = the same metric through the public API with the step's inputs copied host->device from
          pinned memory and the step's results copied back, inside the timed region
roofline: dominant kernel = venom_spmm; achieved = algorithmic FLOPs per launch / mean launch time
          (CUDA events on the launching stream), peak from MEASURED_PEAKS.json
cpu_baseline: the CPU oracle (oracle/) on a bounded sample of the same workload, rank 0, N = 1.
L2: a 512 MiB buffer is written before every timed step (outside the events).
Multi-GPU (torchrun): weak scaling — every rank runs the full workload on its own tokens (the
T/token dimension is the partitioned one); no collective on the data path.
"""
from __future__ import annotations

import argparse
import json
import os
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

# BASELINE configs[1]: the workload `metric` is quoted on at N = 1
WORKLOAD_SETS = {
    "bert_large_ffn_4096tok_64:2:8": ["bert_large_ffn2_1024x4096x4096_64:2:8",
                                      "bert_large_ffn1_4096x1024x4096_64:2:8"],
    "gpt3_ffn_12288x49152x8192_128:2:16": ["gpt3_ffn_12288x49152x8192_128:2:16"],
}
for _k in synth.WORKLOADS:
    WORKLOAD_SETS.setdefault(_k, [_k])
DEFAULT_WORKLOAD = "bert_large_ffn_4096tok_64:2:8"


# measured TMA L2 -> SMEM landing ceiling per SM (GB/s): the SpMM's own steady-state stage rate
# with the L2 idle (8 CTAs: 50 KB per 590 ns per SM, the same as with 148 CTAs, so a per-SM limit;
# profiles/r01_trace_spmm_bert_ffn2_grid8.txt). Higher than tools/microbench_stream.cu's 65 B/ns.
FEED_CEILING_GBPS_PER_SM = 86.8


def useful_flops(w) -> float:
    """2·nnz·T with nnz = R·K·2/M (values are R×K/M×2)."""
    return 2.0 * (w["R"] * (w["K"] // w["M"]) * 2) * w["T"]


def algorithmic_bytes(w) -> float:
    """values + metadata + column_idx + B + C (fp16)."""
    R, K, T, V, M = w["R"], w["K"], w["T"], w["V"], w["M"]
    nnz = R * (K // M) * 2
    return 2 * nnz + nnz / 4 + 4 * (R // V) * (K // M) + 2 * K * T + 2 * R * T


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), d.get("hbm_gbs", 6650.0), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


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
    def __init__(self, name, device, rank, form="auto"):
        import paper_2310_02065_b200 as venom
        self.venom = venom
        self.name = name
        self.w = dict(synth.WORKLOADS[name])
        w = self.w
        sa, sb = synth.seeds(w["cfg"])
        # per-rank tokens (weak scaling): rank r draws its own activations
        self.A = synth.gaussian_device((w["R"], w["K"]), 0.02, synth.F16, sa, device)
        self.B = synth.gaussian_device((w["K"], w["T"]), 1.0, synth.F16, sb + 7919 * rank, device)
        self.bias = synth.gaussian_device((w["R"],), 0.5, synth.F16, sb + 1, device)
        # execution form of the operand: the V:N:M arrays themselves, or the same matrix re-encoded
        # as V:2:4 (reading #18) when that runs faster on B200; either way with the
        # metadata in tensor-core order
        self.expand = (form == "2to4") or (form == "auto" and venom.prefers_2to4(w["R"], w["K"], w["T"], w["V"], w["M"]))
        if self.expand:
            self.x, self.y = venom.compress_2to4(self.A, V=w["V"], M=w["M"], check=True)
        else:
            self.x = venom.compress(self.A, V=w["V"], M=w["M"], check=True)
            self.y = venom.order_metadata(self.x)
        self.C = torch.empty((w["R"], w["T"]), dtype=torch.float16, device=device)
        self.D = torch.empty((w["R"], w["K"]), dtype=torch.float16, device=device)
        self.flops = useful_flops(w)

    def compress(self, A=None):
        """a1-a3 (+ the execution form): one fused kernel for the V:2:4 form, else compress +
        tensor-core ordering of the metadata."""
        w = self.w
        A = self.A if A is None else A
        if self.expand:
            self.venom.compress_2to4(A, V=w["V"], M=w["M"], out=(self.x, self.y))
        else:
            self.venom.compress(A, V=w["V"], M=w["M"], out=self.x)
            self.venom.order_metadata(self.y)

    def spmm(self, B=None, out=None, **kw):
        return self.venom.spmm(self.y, self.B if B is None else B, bias=self.bias,
                               out=self.C if out is None else out, **kw)  # a5-a9

    def decompress(self):
        return self.venom.decompress(self.x, out=self.D)  # a4


def run_gpu(args, ws, rank, local):
    import paper_2310_02065_b200 as venom
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    init_dist(ws, "nccl")
    layers = [Layer(n, device, rank, args.form) for n in WORKLOAD_SETS[args.workload]]
    kw = {}
    if args.tile_t:
        kw["tile_t"] = args.tile_t
    if args.stages:
        kw["stages"] = args.stages
    if args.strategy:
        kw["strategy"] = {"gather": 1, "densek": 2}[args.strategy]
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream(device)

    # the step's kernels as a small DAG over three streams (args.overlap): layer l's compression
    # only feeds layer l's SpMM and decompression, so later layers' compressions run beside the
    # first SpMM and the decompressions (a4) beside the SpMMs; the latency-bound format kernels
    # fill the SMs the persistent SpMM grid leaves idle
    side_c = torch.cuda.Stream(device)
    side_d = torch.cuda.Stream(device)
    comp_done = [torch.cuda.Event() for _ in layers]

    def step(spmm_events=None, part_events=None):
        stream = torch.cuda.current_stream(device)  # the capture stream when recording a graph
        if not args.overlap:
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
            if args.step == "full":
                if part_events is not None:
                    part_events[2].record(stream)
                for L in layers:
                    L.decompress()
                if part_events is not None:
                    part_events[3].record(stream)
            return
        side_c.wait_stream(stream)
        side_d.wait_stream(stream)
        if part_events is not None:
            part_events[0].record(stream)
        layers[0].compress()
        comp_done[0].record(stream)
        with torch.cuda.stream(side_c):
            for i, L in enumerate(layers[1:], 1):
                L.compress()
                comp_done[i].record(side_c)
        if args.step == "full":
            with torch.cuda.stream(side_d):
                if part_events is not None:
                    part_events[2].record(side_d)
                for i, L in enumerate(layers):
                    side_d.wait_event(comp_done[i])
                    L.decompress()
                if part_events is not None:
                    part_events[3].record(side_d)
        if part_events is not None:
            part_events[1].record(stream)
        for i, L in enumerate(layers):
            stream.wait_event(comp_done[i])
            if spmm_events is not None:
                spmm_events[i][0].record(stream)
            L.spmm(**kw)
            if spmm_events is not None:
                spmm_events[i][1].record(stream)
        stream.wait_stream(side_c)
        stream.wait_stream(side_d)

    # [compress_2to4 | compress + order_metadata] + spmm (+ decompress) per layer
    launches_per_step = sum((1 if L.expand else 2) + 1 + int(args.step == "full") for L in layers)
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize(device)
    graph = None
    if args.graph:
        # the whole step as one CUDA graph (both streams): no per-launch CPU/driver gaps
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize(device)
        for _ in range(2):
            flush.zero_()
            graph.replay()
        torch.cuda.synchronize(device)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sp_ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in layers]
             for _ in range(args.steps)]
    pt_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    clocks = ClockSampler(device.index if device.index is not None else 0)
    barrier(ws)
    torch.cuda.synchronize(device)
    # eager pass: per-kernel events (roofline per launch, step breakdown)
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        step(sp_ev[k], pt_ev[k])
        ev[k][1].record(stream)
    torch.cuda.synchronize(device)
    eager_ms = [a.elapsed_time(b) for a, b in ev]
    step_ms = eager_ms
    overlap_spmm_ms = [[a.elapsed_time(b) for a, b in row] for row in sp_ev]
    if args.overlap:
        # the roofline's per-launch SpMM times come from the kernels running alone (serial eager
        # step, as ncu sees them); the overlapped step shares SMs with the format kernels
        ov = args.overlap
        args.overlap = False
        for k in range(args.steps):
            flush.zero_()
            step(sp_ev[k], None)
        torch.cuda.synchronize(device)
        args.overlap = ov
    if graph is not None:
        # timed pass: the captured step replayed K times (L2 flushed before each)
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier(ws)
        torch.cuda.synchronize(device)
        for k in range(args.steps):
            flush.zero_()
            gev[k][0].record(stream)
            graph.replay()
            gev[k][1].record(stream)
        torch.cuda.synchronize(device)
        step_ms = [a.elapsed_time(b) for a, b in gev]
    barrier(ws)
    clk = clocks.stop()
    spmm_ms = [[a.elapsed_time(b) for a, b in row] for row in sp_ev]
    compress_ms = statistics.mean(r[0].elapsed_time(r[1]) for r in pt_ev)
    decompress_ms = statistics.mean(r[2].elapsed_time(r[3]) for r in pt_ev) if args.step == "full" else 0.0
    total_s = max_over_ranks(sum(step_ms) / 1e3, ws, device)
    flops_step = sum(L.flops for L in layers)
    value = aggregate(flops_step * args.steps, ws, total_s) / 1e12
    ms_per_step = total_s * 1e3 / args.steps

    # dominant kernel: venom_spmm (per launch)
    per_launch_ms = [statistics.mean(spmm_ms[k][i] for k in range(args.steps)) for i in range(len(layers))]
    spmm_flops = [L.flops for L in layers]
    achieved = sum(spmm_flops) / (sum(per_launch_ms) / 1e3) / 1e12
    peak_burst, peak_sust, hbm, peak_src = load_peaks()
    traffic, feed = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            tr = json.load(f).get(args.workload)
        if tr:
            traffic = tr.get("dram_bytes_per_launch")
            xb = tr.get("l2_to_smem_bytes_per_launch")
            if xb and len(xb) == len(per_launch_ms):
                # the on-chip feed that binds these kernels: L2 -> SMEM bytes per
                # launch (ncu l1tex__m_xbar2l1tex_read_bytes) over the live launch time, against the
                # measured per-SM landing ceiling × SMs (FEED_CEILING_GBPS_PER_SM)
                ach = sum(xb) / (sum(per_launch_ms) / 1e3) / 1e9
                ceil = FEED_CEILING_GBPS_PER_SM * torch.cuda.get_device_properties(device).multi_processor_count
                feed = {"l2_to_smem_bytes_per_launch": xb, "achieved_GBps": round(ach, 1),
                        "ceiling_GBps": round(ceil, 1), "frac": round(ach / ceil, 4),
                        "ceiling_source": "profiles/r01_trace_spmm_bert_ffn2_grid8.txt (SpMM stage rate per SM, L2 idle)"}
    roofline = {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak_burst, "unit": "TFLOP/s",
                "frac": round(achieved / peak_burst, 4), "traffic": traffic,
                "peak_source": f"{peak_src} bf16 dense burst (fp16 1:1); useful FLOPs of a 2:4 sparse "
                               f"MMA are half its issued FLOPs, so the useful-FLOP peak equals the dense peak",
                "algorithmic_flops_per_launch": [int(x) for x in spmm_flops],
                "mean_launch_ms": [round(x, 5) for x in per_launch_ms],
                "hbm_frac": round(sum(algorithmic_bytes(L.w) for L in layers) / (sum(per_launch_ms) / 1e3) / 1e9 / hbm, 4),
                "feed": feed}

    # cuBLAS dense fp16 baseline at the same shapes (speedup metric)
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    dense = [venom.decompress(L.x) for L in layers]
    cub = []
    for i, L in enumerate(layers):
        ts = []
        for k in range(max(3, args.steps // 2) + 2):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            torch.matmul(dense[i], L.B)
            b.record(stream)
            ts.append((a, b))
        torch.cuda.synchronize(device)
        cub.append(statistics.mean(a.elapsed_time(b) for a, b in ts[2:]))
    speedup = [c / s for c, s in zip(cub, per_launch_ms)]

    # e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        hA = [L.A.cpu().pin_memory() for L in layers]
        hB = [L.B.cpu().pin_memory() for L in layers]
        hC = [torch.empty_like(L.C, device="cpu").pin_memory() for L in layers]
        dA = [torch.empty_like(L.A) for L in layers]
        dB = [torch.empty_like(L.B) for L in layers]

        def e2e_step():
            for i, L in enumerate(layers):
                dA[i].copy_(hA[i], non_blocking=True)
                dB[i].copy_(hB[i], non_blocking=True)
            for i, L in enumerate(layers):
                L.compress(dA[i])
            for i, L in enumerate(layers):
                L.spmm(B=dB[i], **kw)
            if args.step == "full":
                for L in layers:
                    L.decompress()
            for i, L in enumerate(layers):
                hC[i].copy_(L.C, non_blocking=True)
        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize(device)
        barrier(ws)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize(device)
        barrier(ws)
        e2e_s = max_over_ranks(a.elapsed_time(b) / 1e3, ws, device)
        h2d = sum(x.numel() * x.element_size() for x in hA + hB)
        d2h = sum(x.numel() * x.element_size() for x in hC)
        e2e = {"value": round(aggregate(flops_step * args.steps, ws, e2e_s) / 1e12, 3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(layers, budget_s=args.cpu_budget)

    if rank == 0:
        w0 = layers[0].w
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic (seeded; A ~ N(0,0.02^2), B ~ N(0,1), fp16)",
            "config": {"workload": args.workload, "layers": [L.name for L in layers],
                       "V:N:M": f"{w0['V']}:2:{w0['M']}", "tokens_per_gpu": w0["T"],
                       "step": ("compress(+execution form)+spmm" + ("+decompress" if args.step == "full" else "")
                                + " per layer"),
                       "operand_form": ["V:2:4 re-encoding, fused into compress (venom_compress_2to4)" if L.expand
                                        else "V:N:M (+ venom_order_metadata)" for L in layers],
                       "l2": "flushed (512 MiB write) before every timed step", "parallelism": f"T-split x{ws}"},
            "spmm_only": {"tflops": round(achieved, 3), "ms_per_launch": [round(x, 5) for x in per_launch_ms],
                          "ms_per_launch_in_overlapped_step": [round(statistics.mean(r[i] for r in overlap_spmm_ms), 5)
                                                               for i in range(len(layers))]},
            "step_breakdown_ms": {"compress_all_layers": round(compress_ms, 5),
                                  "spmm_all_layers": round(sum(per_launch_ms), 5),
                                  "decompress_all_layers": round(decompress_ms, 5),
                                  "overlapped": ("compress of layers 2.. and decompress (a4) on side streams beside the SpMMs; "
                                                 "compress_all_layers is then the first layer's" if args.overlap else False),
                                  "eager_step_ms": round(statistics.mean(eager_ms), 5),
                                  "timed_as": "CUDA graph replay of the step" if graph is not None else "eager step",
                                  "compress_GBps": round(sum(2 * L.w["R"] * L.w["K"] for L in layers) / compress_ms / 1e6, 1)},
            "speedup_vs_cublas": [round(s, 3) for s in speedup],
            "cublas_ms": [round(c, 5) for c in cub],
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps, "clocks": clk,
        }
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


# ----------------------------------------------------------------------------- CPU oracle
def cpu_baseline(layers, budget_s: float = 12.0, kind: str = "oracle"):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload: full compression of
    every layer plus the SpMM on a column (token) subset sized to ~budget_s."""
    import oracle
    # the oracle works on host copies of the same seeded inputs
    hosts = []
    for L in layers:
        A = L.A.view(torch.int16).cpu().numpy().view(np.uint16) if isinstance(L, Layer) else L["A"]
        B = L.B.view(torch.int16).cpu().numpy().view(np.uint16) if isinstance(L, Layer) else L["B"]
        hosts.append((L.w if isinstance(L, Layer) else L["w"], A, B))
    return time_oracle(hosts, budget_s, kind)


def time_oracle(hosts, budget_s: float, kind: str = "oracle"):
    import oracle
    t0 = time.perf_counter()
    comp = []
    for w, A, B in hosts:
        comp.append(oracle.compress(A, oracle.F16, V=w["V"], M=w["M"]))
    t_comp = time.perf_counter() - t0
    # calibrate columns: one 8-column pass per layer, then scale to the budget
    cols = 8
    t1 = time.perf_counter()
    for (w, A, B), parts in zip(hosts, comp):
        oracle.spmm(*parts, w["R"], w["K"], oracle.F16, w["V"], w["M"], np.ascontiguousarray(B[:, :cols]))
    t_cal = time.perf_counter() - t1
    T = min(min(h[0]["T"], h[2].shape[1]) for h in hosts)  # columns actually available
    cols2 = int(max(8, min(T, cols * max(1.0, (budget_s - t_comp) / max(t_cal, 1e-3)))))
    cols2 -= cols2 % 8
    t2 = time.perf_counter()
    flops = 0.0
    for (w, A, B), parts in zip(hosts, comp):
        oracle.spmm(*parts, w["R"], w["K"], oracle.F16, w["V"], w["M"], np.ascontiguousarray(B[:, :cols2]))
        flops += 2.0 * w["R"] * (w["K"] // w["M"]) * 2 * cols2
    t_sp = time.perf_counter() - t2
    return {"value": flops / (t_sp + t_comp) / 1e12, "unit": UNIT, "cores": oracle.num_threads(),
            "kind": kind,
            "sample": f"full oracle compress of every layer + oracle SpMM on the first {cols2} of "
                      f"{T} token columns per layer ({t_comp:.2f}s compress, {t_sp:.2f}s spmm)",
            "seconds": round(t_comp + t_sp, 3)}


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only)."""
    if rank != 0:
        return
    hosts = []
    for n in WORKLOAD_SETS[args.workload]:
        w = dict(synth.WORKLOADS[n])
        sa, sb = synth.seeds(w["cfg"])
        A = synth.gaussian((w["R"], w["K"]), 0.02, synth.F16, sa)
        B = synth.gaussian((w["K"], min(w["T"], 1024)), 1.0, synth.F16, sb)  # token sample pool
        hosts.append((w, A, B))
    per_step = max(2.0, min(8.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        time_oracle(hosts, per_step)
    vals, secs, last = [], 0.0, None
    for _ in range(args.steps):
        last = time_oracle(hosts, per_step, kind="oracle")
        vals.append(last["value"])
        secs += last["seconds"]
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; same recipe as the GPU arm)",
            "config": {"workload": args.workload, "layers": WORKLOAD_SETS[args.workload],
                       "step": "oracle compress + oracle SpMM on a token sample per layer"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "oracle",
                             "sample": last["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["venom", "reference"], default="venom")
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOAD_SETS))
    ap.add_argument("--step", choices=["full", "spmm"], default="full")
    ap.add_argument("--tile-t", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--strategy", choices=["gather", "densek"], default=None,
                    help="force a venom_spmm strategy (default: the library's cost model)")
    ap.add_argument("--form", choices=["auto", "vnm", "2to4"], default="auto",
                    help="SpMM operand form: V:N:M as compressed, or re-encoded V:2:4 (venom_expand_2to4)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time the eager step instead of its CUDA-graph replay")
    ap.add_argument("--no-overlap", dest="overlap", action="store_false",
                    help="run decompress after the SpMMs on the same stream instead of beside them")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
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
