"""Summarise ncu reports for profiles/: per kernel launch, duration, DRAM bytes, tensor-pipe and
memory throughput; and the launch list share of the step. Usage:
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [workload-key]
  python tools/ncu_summary.py launches <launches.csv> <out.md>"""
import csv, io, json, os, subprocess, sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum"]


def _hbm_peak() -> float:
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"])
    except Exception:
        return 6549.4


HBM_PEAK = _hbm_peak()


def full(rep, out, key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full summary: {os.path.basename(rep)}", "",
             "| kernel | " + " | ".join(KEYS) + " |", "|---" * (len(KEYS) + 1) + "|"]
    traffic = []
    for r in data:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")[:70]
        vals = []
        for k in KEYS:
            vals.append(f"{d.get(k, '-')} {u.get(k, '')}".strip())
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
        try:
            rb = float(d["dram__bytes_read.sum"]); wb = float(d["dram__bytes_write.sum"])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            xb = float(d["l1tex__m_xbar2l1tex_read_bytes.sum"]) * scale.get(u["l1tex__m_xbar2l1tex_read_bytes.sum"], 1)
            traffic.append((rb * scale.get(u["dram__bytes_read.sum"], 1) + wb * scale.get(u["dram__bytes_write.sum"], 1), xb))
        except Exception:
            pass
    # derived: achieved HBM GB/s against the measured peak, L2->SMEM feed, sparse tensor-pipe use
    lines += ["", f"| kernel | duration us | DRAM GB/s | % of HBM peak ({HBM_PEAK} GB/s, MEASURED_PEAKS.json) | "
              "L2->SMEM GB/s | tensor pipe active % |", "|---|---|---|---|---|---|"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
    for r in data:
        d = dict(zip(hdr, r)); uu = dict(zip(hdr, units))
        try:
            t = float(d["gpu__time_duration.sum"]) * scale.get(uu["gpu__time_duration.sum"], 1e-6)
            db = float(d["dram__bytes_read.sum"]) * scale.get(uu["dram__bytes_read.sum"], 1) + \
                float(d["dram__bytes_write.sum"]) * scale.get(uu["dram__bytes_write.sum"], 1)
            xb = float(d["l1tex__m_xbar2l1tex_read_bytes.sum"]) * scale.get(uu["l1tex__m_xbar2l1tex_read_bytes.sum"], 1)
            tp = d.get("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "-")
            lines.append(f"| {d.get('Kernel Name', '?')[:60]} | {t * 1e6:.2f} | {db / t / 1e9:.0f} | "
                         f"{db / t / 1e9 / HBM_PEAK * 100:.1f} | {xb / t / 1e9:.0f} | {tp} |")
        except Exception:
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    if key and traffic:
        p = os.path.join(os.path.dirname(out), "ncu_traffic.json")
        j = json.load(open(p)) if os.path.exists(p) else {}
        j[key] = {"dram_bytes_per_launch": sum(t[0] for t in traffic) / len(traffic),
                  "l2_to_smem_bytes_per_launch": [t[1] for t in traffic], "launches": len(traffic),
                  "source": os.path.basename(rep)}
        json.dump(j, open(p, "w"), indent=1)
    print("\n".join(lines))


def launches(csvf, out):
    txt = open(csvf).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    i_name, i_val, i_metric = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = defaultdict(float); cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= i_val or r[i_metric] != "gpu__time_duration.sum":
            continue
        name = r[i_name].split("(")[0][:80]
        tot[name] += float(r[i_val].replace(",", "")); cnt[name] += 1
    allt = sum(tot.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none): {os.path.basename(csvf)}", "",
             "cold-cache, serialised per-launch times: compare SHARES, not absolutes", "",
             "| kernel | launches | total ns | share |", "|---|---|---|---|"]
    for n, t in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {n} | {cnt[n]} | {t:.0f} | {t / allt:.3f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
