"""cuBLAS fp64 GEMM (via torch.matmul) and torch copy bandwidth on the box: the library reference points."""
import json, torch
def bench(f, reps=10):
    f(); torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); b.synchronize(); best = min(best, a.elapsed_time(b))
    return best
out = {}
for N in (4096, 8192):
    A = torch.randn(N, N, dtype=torch.float64, device="cuda"); B = torch.randn(N, N, dtype=torch.float64, device="cuda")
    ms = bench(lambda: A @ B); out[f"dgemm_{N}_tflops"] = 2 * N**3 / ms / 1e9
for n, p in ((32768, 16), (32768, 64), (16384, 16)):
    M = torch.randn(n, n, dtype=torch.float64, device="cuda"); Y = torch.randn(n, p, dtype=torch.float64, device="cuda")
    ms = bench(lambda: M @ Y); out[f"cublas_MY_n{n}_p{p}_ms"] = ms; out[f"cublas_MY_n{n}_p{p}_gbs"] = 8 * n * n / ms / 1e6
    del M
x = torch.empty(2**29, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
ms = bench(lambda: y.copy_(x)); out["copy_gbs_rw"] = 2 * 8 * 2**29 / ms / 1e6
print(json.dumps(out))
