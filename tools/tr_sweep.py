"""Token-rounding speed sweep of the paper's Fig. 12 on this B200: for each (T, d, n, K)
series and each E, TC vs TR (NR-f) model TFLOPS of the forward (up + down + agg_O) and of the
backward (dH .. agg_dX), plus the padding waste of TC (Fig. 8: rows padded to a 128 multiple).
Writes profiles/<tag>_tr_sweep.md.  Run on the GPU box:  python tools/tr_sweep.py [tag]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SERIES = [  # (T, d, n, K), E values  -- P:2449-2455
    ((16384, 1536, 256, 8), [64, 128, 256, 512]),
    ((16384, 1536, 1024, 2), [16, 32, 64, 128]),
    ((16384, 4096, 512, 8), [64, 128, 256, 512]),
    ((16384, 4096, 1024, 4), [32, 64, 128, 256]),
]
FWD = ("up", "down", "agg_O")


def run(shape, mode):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--shape", ",".join(map(str, shape)),
                          "--mode", mode, "--steps", "10", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"],
                         capture_output=True, text=True, cwd=ROOT).stdout.strip().splitlines()
    d = json.loads(out[-1])
    k = d["kernels"]
    fwd = sum(k[x]["avg_ms"] * k[x]["launches_per_step"] for x in FWD if x in k)
    bwd = sum(v["avg_ms"] * v["launches_per_step"] for x, v in k.items() if x not in FWD and x != "route")
    T, dd, n, E, K = shape
    R = d["rows_routed"]
    f_fwd = 6 * dd * n * R
    f_bwd = 12 * dd * n * R
    return dict(tf=d["value"], fwd=f_fwd / (fwd * 1e-3) / 1e12, bwd=f_bwd / (bwd * 1e-3) / 1e12,
                rows=R, padded=d["rows_padded"], ms=d["ms_per_step"])


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    lines = [f"# Token rounding sweep ({tag}) -- the paper's Fig. 12 configurations on one B200",
             "", "Model TFLOPS = 18 d n R / time (R = routed rows); fwd = up + down + agg_O, bwd = the rest "
             "(router excluded, as in P:1533). TC waste = padded rows of TC that carry no token (Fig. 8).",
             "", "| T, d, n, K | E | TC fwd TF | TR fwd TF | TC bwd TF | TR bwd TF | TC step ms | TR step ms | "
             "TR speed-up | TC padding waste |", "|---|---|---|---|---|---|---|---|---|---|"]
    for (T, d, n, K), Es in SERIES:
        for E in Es:
            shape = (T, d, n, E, K)
            tc, tr = run(shape, "tc"), run(shape, "tr")
            waste = (tc["padded"] - tc["rows"]) / tc["padded"]
            lines.append(f"| {T}, {d}, {n}, {K} | {E} | {tc['fwd']:.0f} | {tr['fwd']:.0f} | {tc['bwd']:.0f} | "
                         f"{tr['bwd']:.0f} | {tc['ms']:.3f} | {tr['ms']:.3f} | {tc['ms'] / tr['ms']:.3f}x | "
                         f"{100 * waste:.1f} % |")
            print(lines[-1], flush=True)
    path = os.path.join(ROOT, "profiles", f"{tag}_tr_sweep.md")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    open(path, "w").write("\n".join(lines) + "\n")
    print("wrote", path)


if __name__ == "__main__":
    main()
