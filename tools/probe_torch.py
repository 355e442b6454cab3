"""Step-0 probe: cuBLAS DGEMM/ZGEMM ceilings via torch (library ceiling, context only)."""
import json, torch, time
def bench(f, reps=5):
    f(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best
out = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    t = bench(lambda: a @ b); out[f"dgemm_{n}_tflops"] = 2 * n**3 / t / 1e12
    a = torch.randn(n, n, dtype=torch.complex128, device="cuda"); b = torch.randn_like(a)
    t = bench(lambda: a @ b); out[f"zgemm_{n}_tflops_8flop"] = 8 * n**3 / t / 1e12
    del a, b
x = torch.empty(2**30 // 8, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
t = bench(lambda: y.copy_(x)); out["copy_gbs"] = 2 * x.numel() * 8 / t / 1e9
print(json.dumps(out))
