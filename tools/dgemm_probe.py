"""cuBLAS DGEMM 8192^3 burst + sustained (same method as MEASURED_PEAKS.json's bf16 entry)."""
import json, time, torch
torch.backends.cuda.matmul.allow_tf32 = False
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
burst = 2 * n**3 / (best * 1e-3) / 1e12
t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; cnt += 1
    if cnt % 8 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sust = 2 * n**3 * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
print(json.dumps({"cublas_dgemm_8192_burst_tflops": round(burst, 3), "cublas_dgemm_8192_sustained_tflops": round(sust, 3)}))
