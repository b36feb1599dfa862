"""bench.py's JSON-line contract.  CPU: the reference arm (the fp64 oracle on the host) on the tiny
config prints one JSON line with the required keys.  GPU: the default arm on the tiny config carries
roofline, cpu_baseline, e2e, gpu_launches and clocks."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_kernel_model_accountings():
    """The tight IO accounting (each gathered tensor read once) never exceeds the paper's (gathered rows
    counted R*d*2), and the two agree for the kernels without a gathered operand."""
    sys.path.insert(0, ROOT)
    import bench
    T, d, n, E, K = 32768, 1536, 256, 128, 8
    R = T * K
    m = bench.kernel_model(T, d, n, E, K, R, R)
    for k, v in m.items():
        assert v["tight"] <= v["paper"], k
    for k in ("down", "dXt", "agg_O", "agg_dX", "route"):
        assert m[k]["tight"] == m[k]["paper"], k
    # FLOPs per routed row: 18 d n over the six GEMMs
    assert sum(m[k]["flops"] for k in ("up", "down", "dH", "dW2", "dXt", "dW1")) == 18 * d * n * R


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "3"])
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("tiny")


@pytest.mark.gpu
def test_default_arm_line_tiny():
    d = _run(["--config", "tiny", "--steps", "5", "--warmup", "3", "--e2e-steps", "3", "--cpu-tokens", "256"])
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm") and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["act_mem_bytes"]["measured"]["held_fwd_to_bwd"] >= d["act_mem_bytes"]["X"]
    # the headline is flushed and uninstrumented; warm and the instrumented breakdown pass sit beside it
    assert d["config"]["l2"].startswith("flushed") and d["warm"]["ms_per_step"] > 0
    assert d["breakdown_pass"]["ms_per_step"] > 0
    # both IO accountings (the tight one never above the paper one) and the spec-peak share
    assert 0 < d["layer_roofline_tight_ms"] <= d["layer_roofline_ms"] * (1 + 1e-9)
    assert d["pct_peak_spec"] == pytest.approx(d["value"] / 2250.0)
    assert "power_w" in d["clocks"] and "power_limit_w" in d["clocks"]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else None
    if peaks and r["bound"] == "tensor":
        assert r["peak"] in (peaks["bf16_tflops"], peaks["bf16_tflops_sustained"])
    if peaks and r["bound"] == "hbm":
        assert r["peak"] == peaks["hbm_gbs"]


@pytest.mark.gpu
@pytest.mark.parametrize("comm", ["nccl", "peer", "peer_sf"])
def test_two_rank_bench_line(comm):
    """The N > 1 path of bench.py (expert parallel, barriers, max-over-ranks timing, rank-0 line) with
    two ranks sharing the one GPU over gloo (SONIC_BENCH_SHARE_GPU; "nccl" then means the
    host-staged DistComm, "peer" the peer-memory kernels over CUDA IPC)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, SONIC_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--config", "tiny", "--steps", "3", "--warmup", "3", "--e2e-steps", "2",
                        "--comm", comm[:4]] + (["--sync-free"] if comm == "peer_sf" else []),
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "ep2"
    ex = d["exchange"]
    assert ex["bytes_out_per_step"] > 0 and ex["layer_roofline_ms_with_exchange"] > ex["nvlink_roofline_ms"] > 0
    assert d["scaling"] == "weak"
