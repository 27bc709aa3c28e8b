"""cuBLAS DGEMM throughput (torch.matmul fp64) on cuda:0 -- FP64 roofline reference."""
import json
import torch

def main():
    out = {}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device="cuda")
        b = torch.randn(n, n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"dgemm_{n}_tflops"] = 2.0 * n ** 3 / best / 1e9
    # batched small GEMM, shape typical of the per-box work (128x192 @ 192x128)
    x = torch.randn(8192, 128, 192, dtype=torch.float64, device="cuda")
    y = torch.randn(8192, 192, 128, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.bmm(x, y)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.bmm(x, y); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out["dgemm_batched_8192x128x192x128_tflops"] = 2.0 * 8192 * 128 * 192 * 128 / best / 1e9
    print(json.dumps(out))

if __name__ == "__main__":
    main()
