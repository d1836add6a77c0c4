"""fp64 GEMM throughput on this GPU: cuBLAS (torch.matmul) for the coarse-factor sizes."""
import torch
torch.backends.cuda.matmul.allow_tf32 = False
for n in (256, 512, 1024, 1700, 3400, 6800, 10000, 20000):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, int(2e11 / (2 * n ** 3)))
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    print(f"n={n:6d}  {t*1e3:9.3f} ms  {2*n**3/t/1e12:6.2f} TFLOP/s fp64 (cuBLAS)")
