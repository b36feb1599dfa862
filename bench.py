#!/usr/bin/env python
"""bench.py -- SonicMoE layer fwd+bwd on B200 through libsonic's C ABI.

One step = sonic_route + sonic_moe_fwd + sonic_moe_bwd over one synthetic microbatch
(all of SURVEY.md section 8(a)'s rows).  Default workload: BASELINE.json configs[1], the
fine-grained 7B-class layer (T=32768, d=1536, n=256, E=128, K=8, token-choice top-K).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 7b|qwen3|...] [--mode tc|tr]
  python bench.py --impl reference ...     # the fp64 CPU oracle on the host cores

N > 1 (torchrun): expert parallelism (paper_2512_14080_b200/ep.py) -- every rank brings its own
T-token microbatch and owns E/N experts; tokens reach their experts' ranks through NCCL all-to-all
(dispatch / combine, forward and backward).  Weak scaling; time = max over ranks; value = model
FLOPs of all ranks' tokens / that time.  `--ep` runs the same EP code at N=1.
Prints ONE JSON line on rank 0.  See DESIGN.md section 7 for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# --mode -> (sonic route mode, oracle mode, oracle rounding); tr = NR-f (the paper's default)
ROUTE_MODES = {"tc": (0, "tc", "nrf"), "tr": (1, "tr", "nrf"), "tr_up": (3, "tr", "up"), "tr_down": (4, "tr", "down"),
               "tr_balance": (5, "tr", "balance"), "tr_sr": (6, "tr", "sr"), "ec": (7, "ec", "nrf"),
               "tr_nrs": (8, "tr", "nrs")}
METRIC = "MoE layer fwd+bwd TFLOPS (% B200 BF16 peak), tokens/s at 1/2/4/8 GPU; act. mem"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


# --------------------------------------------------------------------------- FLOP / byte model
def kernel_model(T, d, n, E, K, R, R_pad, dw=4, fp8_up=False, w1_cached=False, fp8_dxt=False):
    """Algorithmic FLOPs and bytes per launch.

    R = routed rows (T*K under TC, sum f_r under TR).  'paper' bytes count gathered rows at
    R*d*2; 'tight' counts each gathered tensor once.
    """
    b = 2
    W1 = E * d * 2 * n * b
    W2 = E * n * d * b
    ab = 1 if fp8_up else b  # bytes per up-projection operand element (e4m3 with SONIC_F_FP8_UP)
    xb = 1 if fp8_dxt else b  # bytes per dX~ operand element (e4m3 with SONIC_F_FP8_DXT)
    m = {
        "up": dict(flops=4 * R * d * n, paper=R * d * ab + W1 * ab // b + R * 2 * n * b + R * n * b,
                   tight=T * d * ab + W1 * ab // b + R * 2 * n * b + R * n * b),
        "down": dict(flops=2 * R * n * d, paper=R * n * b + W2 + R * d * b, tight=R * n * b + W2 + R * d * b),
        # fused up + down (NEXT-1): A stays on chip, so neither its write nor its read is counted
        "updown": dict(flops=6 * R * d * n, paper=R * d * b + W1 + W2 + R * 2 * n * b + R * d * b,
                       tight=T * d * b + W1 + W2 + R * 2 * n * b + R * d * b),
        "agg_O": dict(flops=0, paper=R * d * b + T * d * b, tight=R * d * b + T * d * b),
        "dH": dict(flops=2 * R * n * d, paper=R * d * b + W2 + 2 * R * 2 * n * b + R * n * b + R * 4,
                   tight=T * d * b + W2 + 2 * R * 2 * n * b + R * n * b + R * 4),
        "dW2": dict(flops=2 * R * n * d, paper=R * n * b + R * d * b + E * n * d * dw,
                    tight=R * n * b + T * d * b + E * n * d * dw),
        "dXt": dict(flops=4 * R * d * n, paper=R * 2 * n * xb + W1 * xb // b + R * d * b,
                    tight=R * 2 * n * xb + W1 * xb // b + R * d * b),
        "dW1": dict(flops=4 * R * d * n, paper=R * d * b + R * 2 * n * b + E * d * 2 * n * dw,
                    tight=T * d * b + R * 2 * n * b + E * d * 2 * n * dw),
        "agg_dX": dict(flops=0, paper=R * d * b + T * d * b, tight=R * d * b + T * d * b),
        "route": dict(flops=0, paper=T * E * 4 + T * K * 8 + R * 12, tight=T * E * 4 + T * K * 8 + R * 12),
        # SONIC_F_FP8_UP: X and W1 read once, their e4m3 copies written (+ scales)
        "quant_fp8": dict(flops=0, paper=T * d * 3 + (0 if w1_cached else E * d * 2 * n * 3),
                          tight=T * d * 3 + (0 if w1_cached else E * d * 2 * n * 3)),
        "dS_reduce": dict(flops=0, paper=R * 8, tight=R * 8),
        # SONIC_F_FP8_DXT: dH read, its e4m3 rows + scales written (+ W1's e4m3 copy unless cached)
        "quant_dh": dict(flops=0, paper=R * 2 * n * 3 + R * 4 + (0 if w1_cached else E * d * 2 * n * 3),
                         tight=R * 2 * n * 3 + R * 4 + (0 if w1_cached else E * d * 2 * n * 3)),
    }
    # bytes written (part of the totals above; reported, not a separate bound: write-only HBM traffic
    # reaches 6.2-7.0 TB/s on B200 with 16/32-byte or TMA stores, tools/hbm_write_probe.cu)
    writes = {"up": R * 2 * n * b + R * n * b, "down": R * d * b, "updown": R * 2 * n * b + R * d * b, "agg_O": T * d * b,
              "dH": R * 2 * n * b + R * n * b + R * 4, "dW2": E * n * d * dw, "dXt": R * d * b,
              "dW1": E * d * 2 * n * dw, "agg_dX": T * d * b, "route": T * K * 8 + R * 12, "dS_reduce": R * 4}
    for k, w in writes.items():
        m[k]["write"] = w
    return m


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,enforced.power.limit,{pw}")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.skip = 0
        self.path = os.path.join("/tmp", f"sonic_clocks_{os.getpid()}.csv")

    @staticmethod
    def power_field(dev):
        # instantaneous board power where the driver has it (power.draw averages over ~1 s, longer than
        # a short timed region); "power.draw" otherwise
        try:
            r = subprocess.run(["nvidia-smi", "-i", str(dev), "--query-gpu=power.draw.instant",
                                "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
            float(r.stdout.strip().splitlines()[0])
            return "power.draw.instant"
        except Exception:
            return "power.draw"

    def start(self):
        try:
            self.fh = open(self.path, "w")
            fields = self.FIELDS.format(pw=self.power_field(self.dev))
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={fields}",
                                          "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # nvidia-smi takes ~0.1-0.5 s to start: wait for its first sample so that the samples that
        # follow fall inside the timed region
        t0 = time.time()
        while time.time() - t0 < 3.0 and self.proc.poll() is None:
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.01)
        self.skip = sum(1 for _ in open(self.path))

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sms, mx, reasons, pw, plim = [], None, set(), [], None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = open(self.path).readlines()
        lines = lines[self.skip:] or lines[-1:]  # drop the idle sample(s) from before the timed region
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
            try:  # board power (instantaneous where available) against the enforced limit
                pw.append(float(parts[8]) if len(parts) > 8 else float(parts[2]))
                plim = float(parts[7]) if len(parts) > 7 else plim
            except ValueError:
                pass
        sms.sort()
        pw.sort()
        med = sms[len(sms) // 2] if sms else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sms),
                "power_w": pw[len(pw) // 2] if pw else None, "power_w_max": pw[-1] if pw else None,
                "power_limit_w": plim}


# --------------------------------------------------------------------------- CPU oracle leg
def oracle_sample(cfg, mode, seed, T_sample, m_tile=128):
    """The fp64 oracle as it stands on a bounded sample: the first T_sample tokens of the
    workload (route + fwd + bwd).  Returns (model FLOPs processed, seconds, threads)."""
    import numpy as np
    import torch
    from oracle import moe_oracle as om
    from paper_2512_14080_b200.inputs import make_inputs
    c = dict(cfg)
    c["T"] = T_sample
    inp = make_inputs(**c, seed=seed, device="cpu")
    f64 = lambda t: t.float().numpy().astype(np.float64)
    X, W1, W2, dO, S = f64(inp.X), f64(inp.W1), f64(inp.W2), f64(inp.dO), inp.S.numpy()
    t0 = time.perf_counter()
    _, omode, rounding = ROUTE_MODES[mode]
    rt = om.route(S, c["K"], mode=omode, m_tile=m_tile, rounding=rounding)
    om.forward(X, W1, W2, rt)
    om.backward(dO, X, W1, W2, rt)
    dt = time.perf_counter() - t0
    flops = 18 * c["d"] * c["n"] * rt.R
    try:  # the BLAS pool numpy actually used
        from threadpoolctl import threadpool_info
        threads = max([p.get("num_threads", 1) for p in threadpool_info() if p.get("user_api") == "blas"] or [1])
    except Exception:
        threads = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    return flops, dt, threads


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    T_s = args.ref_tokens
    for _ in range(args.warmup):
        oracle_sample(cfg, args.mode, 0, T_s, args.m_tile)
    tot_f, tot_t, thr = 0, 0.0, 1
    for i in range(args.steps):
        f, t, thr = oracle_sample(cfg, args.mode, i, T_s, args.m_tile)
        tot_f += f
        tot_t += t
    v = tot_f / tot_t / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, cfg),
        "cpu_baseline": {"value": v, "unit": "TFLOPS", "cores": thr, "kind": "oracle",
                         "sample": f"first {T_s} tokens of the workload per step (route+fwd+bwd, fp64 numpy)"},
        "e2e": {"value": v, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, cfg):
    return {"workload": f"{args.config}: T={cfg['T']} d={cfg['d']} n={cfg['n']} E={cfg['E']} K={cfg['K']} "
                        f"route={args.mode}",
            "T": cfg["T"], "d": cfg["d"], "n": cfg["n"], "E": cfg["E"], "K": cfg["K"], "route": args.mode,
            "parallelism": f"ep{args.gpus}" if (args.gpus > 1 or getattr(args, "ep", False)) else "single",
            **({"cuda_graph": "one step captured and replayed"} if getattr(args, "graph", False) else {}),
            **({"ep_exchange": ("peer-memory kernels (CUDA IPC)" + (", host-sync-free (device offsets, capacity "
                                                                    "2*T*K pairs)" if getattr(args, "sync_free", False)
                                                                    else "")) if args.comm == "peer"
                else "NCCL all-to-all-v" + (", chunked dispatch (self block first)" if getattr(args, "chunked", False)
                                            else "")}
               if (args.gpus > 1 or getattr(args, "ep", False)) else {}),
            **({"dW": "bf16 (SONIC_F_DW_BF16)"} if getattr(args, "dw_bf16", False) else {}),
            **({"updown": "fused kernel (SONIC_F_FUSED_UPDOWN)"} if getattr(args, "fuse", False) else {}),
            **({"up_proj": "e4m3 operands (SONIC_F_FP8_UP), everything else bf16" +
                          ("; W1's e4m3 copy cached across steps (SONIC_F_FP8_W1_CACHED)"
                           if getattr(args, "fp8_w1_cached", False) else "")} if getattr(args, "fp8_up", False)
               else {}),
            **({"dXt": "e4m3 operands (SONIC_F_FP8_DXT: dH x the forward's W1 column scales, per-row quantised)"}
               if getattr(args, "fp8_dxt", False) else {}),
            **({"m_tile": args.m_tile} if getattr(args, "m_tile", 128) != 128 else {}),
            "l2": ("flushed before every timed step (memset of 2x L2 outside the step's event pair); warm "
                   "back-to-back number in `warm`") if getattr(args, "l2_flush", False) else
                  "not flushed: per-step working set (X, W1, W2, H, Y, dX~, ...) is several GB >> 126 MB L2"}


# --------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="sonic", choices=["sonic", "reference"])
    ap.add_argument("--config", default="7b")
    ap.add_argument("--shape", default="", help="T,d,n,E,K: a custom workload instead of --config (sweeps)")
    ap.add_argument("--mode", default="tc", choices=list(ROUTE_MODES))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--ref-tokens", type=int, default=1024)
    ap.add_argument("--cpu-tokens", type=int, default=8192)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--breakdown", default="", help="write the per-kernel table to this JSON file")
    ap.add_argument("--ep", action="store_true", help="expert-parallel path even at N=1 (always on for N>1)")
    ap.add_argument("--m-tile", type=int, default=128, choices=[128, 256],
                    help="token-rounding tile (256 = the 2-CTA pair's M tile: no half-empty pairs)")
    ap.add_argument("--dw-bf16", action="store_true", help="SONIC_F_DW_BF16: weight gradients stored as bf16")
    ap.add_argument("--fp8-up", action="store_true",
                    help="SONIC_F_FP8_UP: the up-projection on e4m3 operands (NEXT-4; not the bf16 headline)")
    ap.add_argument("--fp8-dxt", action="store_true",
                    help="SONIC_F_FP8_DXT: dX~ on e4m3 operands (NEXT-4, DESIGN Q25; not the bf16 headline)")
    ap.add_argument("--fp8-w1-cached", action="store_true",
                    help="with --fp8-up: SONIC_F_FP8_W1_CACHED after the first step (W1's e4m3 copy reused, as in the "
                         "micro-batches of a gradient-accumulation step)")
    ap.add_argument("--fuse", action="store_true",
                    help="SONIC_F_FUSED_UPDOWN: the fused up/down kernel (A kept on chip) instead of two kernels")
    ap.add_argument("--no-l2-flush", dest="l2_flush", action="store_false",
                    help="time the K steps back to back without flushing L2 (the primary number flushes)")
    ap.add_argument("--sustain-s", type=float, default=0.0,
                    help="also run the step back to back for this many seconds (sustained / power-capped regime)")
    ap.add_argument("--sync-free", action="store_true",
                    help="with --comm peer: the host-sync-free exchange (offsets read on the device, NEXT-2)")
    ap.add_argument("--chunked", action="store_true",
                    help="EP (NCCL exchange): chunked dispatch -- the self block's GEMMs run while the remote "
                         "blocks are exchanged (NEXT-2)")
    ap.add_argument("--graph", action="store_true",
                    help="capture one step in a CUDA graph and replay it in the timed passes (needs a step "
                         "without host synchronisation: the single-GPU path, or --comm peer --sync-free)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "peer"],
                    help="EP exchange: NCCL all-to-all-v, or libsonic's peer-memory kernels (CUDA IPC / NVLink)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2512_14080_b200.inputs import CONFIGS
    if args.shape:
        T_, d_, n_, E_, K_ = (int(v) for v in args.shape.split(","))
        cfg = dict(T=T_, d=d_, n=n_, E=E_, K=K_)
        args.config = f"custom_{args.shape.replace(',', 'x')}"
    else:
        cfg = CONFIGS[args.config]

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2512_14080_b200 import sonic
    from paper_2512_14080_b200.inputs import make_inputs

    # test-only: several ranks sharing one GPU (the single-GPU box) exercise the N > 1 code path over
    # gloo; the exchange is then the host-staged DistComm or the peer-memory kernels, never NCCL
    share_gpu = os.environ.get("SONIC_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if os.environ.get("SONIC_L2_PERSIST_MB"):  # experiment: L2 set-aside for evict_last lines
        import ctypes
        rt_ = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
        if rt_ is not None:
            mb = int(os.environ["SONIC_L2_PERSIST_MB"])
            st = rt_.cudaDeviceSetLimit(ctypes.c_int(6), ctypes.c_size_t(mb << 20))  # cudaLimitPersistingL2CacheSize
            got = ctypes.c_size_t(0)
            rt_.cudaDeviceGetLimit(ctypes.byref(got), ctypes.c_int(6))
            mx = ctypes.c_int(0)
            rt_.cudaDeviceGetAttribute(ctypes.byref(mx), ctypes.c_int(108), ctypes.c_int(local))  # MaxPersistingL2CacheSize
            print(f"[l2 persist] set {mb} MB -> status {st}, limit {got.value >> 20} MB (max {mx.value >> 20} MB)",
                  file=sys.stderr)
    if world > 1:
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    T, d, n, E, K = cfg["T"], cfg["d"], cfg["n"], cfg["E"], cfg["K"]
    mode = ROUTE_MODES[args.mode][0]
    desc = sonic.make_desc(T, d, n, E, K, mode=mode, m_tile=args.m_tile,
                           flags=(sonic.SONIC_F_DW_BF16 if args.dw_bf16 else 0) |
                           (sonic.SONIC_F_FUSED_UPDOWN if args.fuse else 0) |
                           (sonic.SONIC_F_FP8_UP if args.fp8_up else 0) |
                           (sonic.SONIC_F_FP8_DXT if args.fp8_dxt else 0))
    use_ep = args.ep or world > 1
    if not use_ep:
        # ---- one GPU, all experts local: route + fwd + bwd through the C ABI
        inp = make_inputs(**cfg, seed=args.seed + rank, device=dev)
        X, S, dOin, W1, W2 = inp.X, inp.S, inp.dO, inp.W1, inp.W2
        rows = sonic.sonic_rows_max(desc)
        rt = sonic.alloc_routing(desc, dev)
        ws_r = torch.empty(max(256, sonic.sonic_route_workspace_size(desc)), dtype=torch.uint8, device=dev)
        ws_f = torch.empty(max(256, sonic.sonic_fwd_workspace_size(desc)), dtype=torch.uint8, device=dev)
        ws_b = torch.empty(max(256, sonic.sonic_bwd_workspace_size(desc)), dtype=torch.uint8, device=dev)
        # outputs double-buffered so the e2e pipeline can read step i's O/dX while step i+1 runs
        Obuf = [torch.empty(T, d, dtype=torch.bfloat16, device=dev) for _ in range(2)]
        dXbuf = [torch.empty(T, d, dtype=torch.bfloat16, device=dev) for _ in range(2)]
        H = torch.empty(rows, 2 * n, dtype=torch.bfloat16, device=dev)
        wdt = torch.bfloat16 if args.dw_bf16 else torch.float32
        dW1 = torch.empty(E, d, 2 * n, dtype=wdt, device=dev)
        dW2 = torch.empty(E, n, d, dtype=wdt, device=dev)
        dS = torch.empty(rows, dtype=torch.float32, device=dev)

        # --fp8-w1-cached: the first forward quantises W1 into ws_f, later ones reuse it
        desc_f = [desc]
        desc_b = [desc]

        def run(Xa, Sa, dOa, slot=0):
            O, dX = Obuf[slot], dXbuf[slot]
            sonic.sonic_route(desc, Sa, rt, ws_r)
            sonic.sonic_moe_fwd(desc_f[0], Xa, W1, W2, rt, O, H, ws_f)
            if args.fp8_w1_cached and not (desc_f[0].flags & sonic.SONIC_F_FP8_W1_CACHED):
                desc_f[0] = sonic.make_desc(T, d, n, E, K, mode=mode, m_tile=args.m_tile,
                                            flags=desc.flags | sonic.SONIC_F_FP8_W1_CACHED)
            sonic.sonic_moe_bwd(desc_b[0], dOa, Xa, H, W1, W2, rt, dX, dW1, dW2, dS, ws_b)
            desc_b[0] = desc_f[0]  # the bwd workspace's e4m3 W1 copy is valid from the second step on
            return O, dX

        def routed_rows():
            return int(rt.offsets[E].item()), int(rt.pad_offsets[E].item())

        def local_model(R, R_pad):
            return kernel_model(T, d, n, E, K, R, R_pad, dw=2 if args.dw_bf16 else 4, fp8_up=args.fp8_up,
                                w1_cached=args.fp8_w1_cached, fp8_dxt=args.fp8_dxt)
    else:
        # ---- expert parallelism over the `world` GPUs (NCCL all-to-all), weak scaling: every rank
        #      brings its own T tokens and owns E/world experts (paper_2512_14080_b200/ep.py)
        from paper_2512_14080_b200 import ep
        from paper_2512_14080_b200.inputs import make_expert_weights, make_token_inputs
        G = world
        L = E // G
        X, dOin, S = make_token_inputs(T, d, E, seed=args.seed + 17 * rank, device=dev)
        W1, W2 = make_expert_weights(rank * L, (rank + 1) * L, d, n, seed=args.seed, device=dev)
        if args.comm == "peer":
            comm = ep.PeerComm(G, T, d, L, [rank], sync_free=args.sync_free)
        else:
            comm = ep.DistComm() if world > 1 else ep.SimComm(1)
        rk = ep.EPRank(T, d, n, E, K, G, rank, W1, W2, mode=mode)

        def run(Xa, Sa, dOa, slot=0):
            (Oa,) = ep.ep_forward([rk], comm, [Xa], [Sa], chunked=args.chunked)
            ((dXa, _),) = ep.ep_backward([rk], comm, [dOa])
            return Oa, dXa

        def routed_rows():
            rt0 = rk.ctx["rt"]
            return int(rt0.offsets[E].item()), int(rt0.pad_offsets[E].item())

        def local_model(R, R_pad):
            # the GEMMs run on the R_in rows this rank received, over its L experts (GIVEN routing)
            R_in = rk.ctx["R_in"]
            if R_in == 0:
                return kernel_model(1, d, n, L, L, 0, 0)
            if rk.ctx.get("chunked"):
                # chunked dispatch: one launch of each kernel per chunk -- the per-launch model is the
                # chunks' total work over the chunk count (an average, like the measured per-launch time)
                ch = rk.ctx["chunks"]
                Rr = sum(int(c["lrt"].offsets[L].item()) for c in ch)
                Rp = sum(int(c["lrt"].pad_offsets[L].item()) for c in ch)
                m = kernel_model(R_in, d, n, L, L, Rr, Rp)
                return {k: {q: v / len(ch) for q, v in mm.items()} for k, mm in m.items()}
            lrt = rk.ctx["lrt"]
            return kernel_model(R_in, d, n, L, L, int(lrt.offsets[L].item()), int(lrt.pad_offsets[L].item()))

    def step_eager():
        run(X, S, dOin)

    step = step_eager
    for _ in range(max(args.warmup, 1)):  # >= 1 untimed step so R is known below
        step()
    torch.cuda.synchronize()
    graph = None
    if args.graph:
        # the whole step as one CUDA graph (launch overhead and Python out of the timed region); the
        # per-kernel breakdown pass below stays eager (its events are recorded by the library calls)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step_eager()
        torch.cuda.synchronize()
        step = graph.replay
        step()
        torch.cuda.synchronize()
    R, R_pad = routed_rows()
    flops_step = 18 * d * n * R
    flops_all = flops_step
    if world > 1:
        ft = torch.tensor([float(flops_step)], device=dev, dtype=torch.float64)
        dist.all_reduce(ft)
        flops_all = float(ft.item())

    # ---- device-timed region: inputs resident in HBM, no instrumentation inside it
    # Primary number: L2 flushed before every step (a write of 2x the L2 size, outside
    # the step's own event pair); `warm` beside it: the same K steps back to back, L2 not flushed.
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(max(2 * l2_bytes, 1 << 20), dtype=torch.uint8, device=dev) if args.l2_flush else None

    def timed_pass(flush, profile=False):
        clocks = ClockSampler(local)
        sonic.sonic_profile_enable(profile)
        sonic.sonic_profile_collect()
        sonic.LAUNCHES[0] = 0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clocks.start()
        if flush:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for a, b in evs:
                flush_buf.zero_()
                a.record()
                step()
                b.record()
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs)
        else:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            for _ in range(args.steps):
                step()
            ev1.record()
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
        clk = clocks.stop()
        if world > 1:
            dist.barrier()
        sonic.sonic_profile_enable(False)
        recs = sonic.sonic_profile_collect()
        launches = sonic.LAUNCHES[0]
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, clk, recs, launches

    ms, clk, _, gpu_launches = timed_pass(args.l2_flush)
    ms_step = ms / args.steps
    value = flops_all / (ms_step * 1e-3) / 1e12
    ms_w, clk_w, _, _ = timed_pass(False) if args.l2_flush else (ms, clk, None, None)
    warm = {"ms_per_step": ms_w / args.steps, "value": flops_all / (ms_w / args.steps * 1e-3) / 1e12,
            "clocks": clk_w, "l2": "not flushed (steps back to back)"}
    # per-kernel breakdown: a second pass of the same K steps with every launch bracketed by CUDA
    # events on its own stream (sonic_profile_*), so the headline above carries no instrumentation
    step = step_eager  # the breakdown pass: per-launch events need the eager calls
    ms_p, clk_p, recs, _ = timed_pass(False, profile=True)
    step = graph.replay if graph is not None else step_eager
    sustained = None
    if args.sustain_s > 0:
        # seconds-long back-to-back run: the regime the sustained (power-capped) peak describes
        n_sus = 0
        clocks = ClockSampler(local)
        torch.cuda.synchronize()
        clocks.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.time()
        while time.time() - t0 < args.sustain_s:
            for _ in range(20):
                step()
            n_sus += 20
            e1.record()
            e1.synchronize()
        e1.record()
        torch.cuda.synchronize()
        sus_ms = e0.elapsed_time(e1) / n_sus
        sustained = {"seconds": args.sustain_s, "steps": n_sus, "ms_per_step": sus_ms,
                     "value": flops_all / (sus_ms * 1e-3) / 1e12, "clocks": clocks.stop()}

    # ---- per-kernel breakdown and roofline of the dominant kernel
    peaks = load_peaks()
    model = local_model(R, R_pad)
    agg = {}
    for name, t in recs:
        a = agg.setdefault(name, [0.0, 0])
        a[0] += t
        a[1] += 1
    # Tensor peak for the roofline: the burst figure (MEASURED_PEAKS bf16_tflops) -- the K timed steps
    # are a short region; the sustained figure belongs to the seconds-long `sustained` run (--sustain-s)
    # and is reported beside it as frac_vs_sustained
    tf_peak = peaks["bf16_tflops"]
    tf_sus = peaks["bf16_tflops_sustained"]
    peak_choice = "bf16_tflops (burst): K-step timed region; frac_vs_sustained uses bf16_tflops_sustained"
    bw_peak = peaks["hbm_gbs"]
    kernels = {}
    for name, (tot, cnt) in agg.items():
        avg = tot / cnt
        mm = model.get(name, dict(flops=0, paper=0, tight=0, write=0))
        # the e4m3 up-projection is held to the fp8 peak: the measured bf16 peak x 2 (the guide's nominal
        # dense fp8 : bf16 ratio, 4.5 : 2.25 PFLOP/s)
        kpeak = tf_peak * (2.0 if ((args.fp8_up and name == "up") or (args.fp8_dxt and name == "dXt")) else 1.0)
        t_tensor = mm["flops"] / (kpeak * 1e12) * 1e3
        t_hbm = mm["paper"] / (bw_peak * 1e9) * 1e3  # all algorithmic bytes at the measured copy rate
        kernels[name] = dict(avg_ms=avg, launches_per_step=cnt / args.steps, share=tot / ms_p if ms_p else None,
                             tflops=mm["flops"] / (avg * 1e-3) / 1e12 if mm["flops"] else 0.0,
                             gbs_paper=mm["paper"] / (avg * 1e-3) / 1e9, gbs_tight=mm["tight"] / (avg * 1e-3) / 1e9,
                             bound="tensor" if t_tensor >= t_hbm else "hbm",
                             roofline_ms=max(t_tensor, t_hbm), frac=max(t_tensor, t_hbm) / avg if avg else None,
                             roofline_ms_tight=max(t_tensor, mm["tight"] / (bw_peak * 1e9) * 1e3),
                             tensor_peak=kpeak)
    dom = max(kernels, key=lambda k: kernels[k]["avg_ms"] * kernels[k]["launches_per_step"]) if kernels else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if dom and os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{args.config}/{args.mode}/{dom}")
    roof = None
    if dom:
        k = kernels[dom]
        if k["bound"] == "tensor":
            kp = k["tensor_peak"]
            roof = {"kernel": dom, "bound": "tensor", "achieved": k["tflops"], "peak": kp, "unit": "TFLOP/s",
                    "frac": k["tflops"] / kp, "frac_vs_sustained": k["tflops"] / (tf_sus * kp / tf_peak), "traffic": traffic,
                    "algorithmic_per_launch": model[dom]["flops"], "peak_source": peaks["source"] + " " + peak_choice}
        else:
            roof = {"kernel": dom, "bound": "hbm", "achieved": k["gbs_paper"], "peak": bw_peak, "unit": "GB/s",
                    "frac": k["gbs_paper"] / bw_peak, "traffic": traffic,
                    "algorithmic_per_launch": model[dom]["paper"], "peak_source": peaks["source"] + " hbm_gbs"}
    layer_roof_ms = sum(kernels[k]["roofline_ms"] * kernels[k]["launches_per_step"] for k in kernels)
    # SURVEY 8(d)'s second IO accounting: each gathered tensor read once (the L2-ideal gather)
    layer_roof_tight_ms = sum(kernels[k]["roofline_ms_tight"] * kernels[k]["launches_per_step"] for k in kernels)
    exchange = None
    if use_ep:
        # NVLink bytes this rank moves per step (rows to / from the OTHER ranks): forward X rows +
        # gates out, Y partial sums back; backward dO rows out, dX~ partial sums + dS back
        G_ = world
        sc, rc = rk.ctx["counts"], rk.ctx["recv_counts"]
        if sc is None:  # host-sync-free exchange: read the count matrix now, outside the timed region
            Mfull = comm.regions[0].view(comm.lay["counts"], (G_, comm.NB * G_), torch.int32).cpu().tolist()
            sc = Mfull[rank][:G_]
            rc = [Mfull[s_][rank] for s_ in range(G_)]
        s_off = sum(c for g, c in enumerate(sc) if g != rank)
        r_off = sum(c for g, c in enumerate(rc) if g != rank)
        L_ = E // G_
        out_b = s_off * (2 * d * 2 + L_ * 4) + r_off * (2 * d * 2 + L_ * 4)
        in_b = r_off * (2 * d * 2 + L_ * 4) + s_off * (2 * d * 2 + L_ * 4)
        nvl_gbs = 900.0  # NVLink 5 per direction per GPU (nominal)
        nvl_ms = max(out_b, in_b) / (nvl_gbs * 1e9) * 1e3
        exchange = {"bytes_out_per_step": out_b, "bytes_in_per_step": in_b, "nvlink_gbs_nominal": nvl_gbs,
                    "nvlink_roofline_ms": nvl_ms,
                    "layer_roofline_ms_with_exchange": layer_roof_ms + nvl_ms}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # Pipelined over three streams, each step's transfers inside the timed region: the H2D of
        # step i+1 and the D2H of step i-1 overlap the compute of step i (inputs and outputs are
        # double-buffered; PCIe is full duplex).
        Xh = X.cpu().pin_memory()
        Sh = S.cpu().pin_memory()
        dOh = dOin.cpu().pin_memory()
        Oh = [torch.empty(T, d, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
        dXh = [torch.empty(T, d, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
        Xd = [torch.empty_like(X) for _ in range(2)]
        Sd = [torch.empty_like(S) for _ in range(2)]
        dOd = [torch.empty_like(dOin) for _ in range(2)]
        s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()
        ev_in = [ev(), ev()]    # inputs of slot b landed
        ev_cmp = [ev(), ev()]   # compute of slot b done (inputs free, outputs ready)
        ev_out = [ev(), ev()]   # D2H of slot b done (outputs free)
        for b in range(2):      # all slots start free
            for e_ in (ev_cmp[b], ev_out[b]):
                e_.record(s_cmp)

        def step_e2e(i):
            b = i & 1
            with torch.cuda.stream(s_in):
                s_in.wait_event(ev_cmp[b])
                Xd[b].copy_(Xh, non_blocking=True)
                Sd[b].copy_(Sh, non_blocking=True)
                dOd[b].copy_(dOh, non_blocking=True)
                ev_in[b].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in[b])
                s_cmp.wait_event(ev_out[b])
                Od, dXd = run(Xd[b], Sd[b], dOd[b], b)
                Od.record_stream(s_out)
                dXd.record_stream(s_out)
                ev_cmp[b].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[b])
                Oh[b].copy_(Od, non_blocking=True)
                dXh[b].copy_(dXd, non_blocking=True)
                ev_out[b].record(s_out)

        step_e2e(0)
        step_e2e(1)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_in)
        for i in range(args.e2e_steps):
            step_e2e(i)
        s_in.wait_stream(s_out)
        e1.record(s_in)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e_step = ems / args.e2e_steps
        e2e = {"value": flops_all / (e_step * 1e-3) / 1e12, "unit": "TFLOPS",
               "h2d_bytes_per_step": Xh.numel() * 2 + Sh.numel() * 4 + dOh.numel() * 2,
               "d2h_bytes_per_step": Oh[0].numel() * 2 + dXh[0].numel() * 2, "ms_per_step": e_step,
               "pipelined": "H2D(i+1) | compute(i) | D2H(i-1) on three streams"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        f, t, thr = oracle_sample(cfg, args.mode, args.seed, args.cpu_tokens, args.m_tile)
        cpu = {"value": f / t / 1e12, "unit": "TFLOPS", "cores": thr, "kind": "oracle",
               "sample": f"first {args.cpu_tokens} of {T} tokens (route+fwd+bwd in fp64 numpy), {t:.1f} s"}

    meta_bytes = sum(sonic.sonic_routing_sizes(desc).values())
    act = {"X": T * d * 2, "H": R_pad * 2 * n * 2, "metadata": meta_bytes,
           "paper_formula_2Td_4TKn": 2 * T * d + 4 * T * K * n}
    act["total"] = act["X"] + act["H"] + act["metadata"]
    if not use_ep:
        # the allocations the step actually holds from the forward to the backward (routing tensors +
        # the H cache; X is the caller's), and the transient workspaces (A, Y in fwd; dH, A', dX~ in bwd)
        held = sum(t.numel() * t.element_size() for t in rt.tensors.values()) + H.numel() * H.element_size()
        act["measured"] = {"held_fwd_to_bwd": held + X.numel() * X.element_size(),
                           "fwd_workspace": ws_f.numel(), "bwd_workspace": ws_b.numel(),
                           "peak_allocated": torch.cuda.max_memory_allocated(dev)}
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": ("bf16+e4m3(" + ",".join(k for k, f in (("up-proj", args.fp8_up),
                                                                               ("dX~", args.fp8_dxt)) if f) + ")")
        if (args.fp8_up or args.fp8_dxt) else "bf16", "data": "synthetic",
        "config": workload_config(args, cfg),
        "pct_peak": value / world / peaks["bf16_tflops"],
        "pct_peak_sustained": value / world / peaks["bf16_tflops_sustained"],
        "tokens_per_s": T * world / (ms_step * 1e-3),
        "model_flops_per_step": flops_all, "rows_routed": R, "rows_padded": R_pad,
        "layer_roofline_ms": layer_roof_ms, "layer_roofline_frac": layer_roof_ms / ms_step,
        "layer_roofline_tight_ms": layer_roof_tight_ms, "layer_roofline_tight_frac": layer_roof_tight_ms / ms_step,
        # against the nominal dense bf16 figure (2.25 PFLOP/s, B200_PROFILING.md) beside the measured peaks
        "pct_peak_spec": value / world / 2250.0,
        # the same metric without sonic_route (the paper's bounds exclude the router)
        "value_excl_route": (flops_all / ((ms_step - kernels["route"]["avg_ms"] * kernels["route"]["launches_per_step"])
                                          * 1e-3) / 1e12) if "route" in kernels else None,
        "act_mem_bytes": act, "warm": warm, "sustained": sustained,
        "breakdown_pass": {"ms_per_step": ms_p / args.steps, "clocks": clk_p,
                           "note": "per-kernel events on (sonic_profile_enable); kernels/roofline come from it"},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches,
        "clocks": clk, "kernels": kernels, "exchange": exchange, "peaks": {k: peaks.get(k) for k in ("hbm_gbs", "bf16_tflops",
                                                                                "bf16_tflops_sustained", "source")},
    }
    if args.breakdown:
        json.dump(line, open(args.breakdown, "w"), indent=1)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
