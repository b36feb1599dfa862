"""Summarise ncu outputs into committed, judge-readable files under profiles/.

usage: python tools/ncu_summary.py <round-tag> <launches.csv> <name=report.ncu-rep> ...
Writes profiles/ncu_summary_<tag>.md, profiles/launches_<tag>.csv (per-launch device times of
one step) and updates profiles/traffic.json (DRAM bytes per launch of each profiled GEMM,
read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_dim_x", "cluster x"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
    return f * scale


def main():
    tag, launches = sys.argv[1], sys.argv[2]
    reps = dict(a.split("=", 1) for a in sys.argv[3:])
    lines = [f"# ncu summary, round {tag}", "",
             "7B config (T=32768, d=1536, n=256, E=128, K=8, TC), one step after one warm-up step, "
             "`ncu --set full --clock-control none` (cold caches, replayed: compare shares, not absolutes).", ""]
    # launch list
    rows = list(csv.reader(open(launches)))
    hdr = None
    recs = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                recs.append((d["Kernel Name"], float(d["Metric Value"].replace(",", "")), d["Metric Unit"]))
    recs = [r for r in recs if "sonic" in r[0]]  # our kernels (drop torch's input generation)
    step = recs[len(recs) // 2:]  # second (timed) step
    tot = sum(v for _, v, _ in step)
    with open(os.path.join(ROOT, "profiles", f"launches_{tag}.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "duration_ns", "share_of_step"])
        for k, v, u in step:
            ns = v * (1000 if u in ("usecond", "us") else 1)
            w.writerow([k[:90], f"{ns:.0f}", f"{v / tot:.4f}"])
    lines += ["## Launch list of one step (ncu gpu__time_duration, serialised)", "",
              "| kernel | µs | share |", "|---|---|---|"]
    for k, v, u in step:
        us = v / 1000 if u in ("nsecond", "ns") else v
        lines.append(f"| `{k[:70]}` | {us:.1f} | {v / tot:.3f} |")
    lines.append("")
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for name, rep in reps.items():
        m = raw(rep)
        lines += [f"## {name}: `{m.get('Kernel Name', ('?',))[0][:100]}`", "", "| metric | value |", "|---|---|"]
        for key, label in METRICS:
            if key in m:
                v, u = m[key]
                lines.append(f"| {label} (`{key}`) | {v} {u} |")
        if "dram__bytes_read.sum" in m and "dram__bytes_write.sum" in m:
            b = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
            traffic[f"7b/tc/{name}"] = b
            lines.append(f"| DRAM traffic per launch (read+write) | {b / 1e6:.1f} MB |")
        lines.append("")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    open(os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.md"), "w").write("\n".join(lines) + "\n")
    print(f"wrote profiles/ncu_summary_{tag}.md")


if __name__ == "__main__":
    main()
