"""cuBLAS (torch.bmm) reference rates on the 7B layer's per-expert GEMM shapes (E=128 batched,
2048 rows per expert): what a vendor dense GEMM reaches on the same problem sizes (no gather,
no fused epilogue).  Context for the grouped GEMMs' roofline fractions."""
import torch

E, Rm, d, n = 128, 2048, 1536, 256
shapes = {
    "up    (Rm x d) @ (d x 2n)": (Rm, d, 2 * n),
    "down  (Rm x n) @ (n x d)": (Rm, n, d),
    "dH    (Rm x d) @ (d x n)": (Rm, d, n),
    "dXt   (Rm x 2n) @ (2n x d)": (Rm, 2 * n, d),
    "dW2   (n x Rm) @ (Rm x d)": (n, Rm, d),
    "dW1   (d x Rm) @ (Rm x 2n)": (d, Rm, 2 * n),
}
for name, (M, K, N) in shapes.items():
    a = torch.randn(E, M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(E, K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = torch.bmm(a, b)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    it = 20
    for _ in range(it):
        c = torch.bmm(a, b)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / it
    print(f"{name:30s} {ms * 1e3:8.1f} us  {2 * E * M * K * N / ms / 1e9:8.1f} TFLOPS")
