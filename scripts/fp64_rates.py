"""Measure fp64 dense rates on this GPU (cuBLAS DGEMM, cuSOLVER getrf/getrs via
torch) at the block sizes the local-solve build uses.  Diagnostic only."""
import torch

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3

d = "cuda"
for n in (8192, 4096, 2048, 1024, 512):
    a = torch.randn(n, n, dtype=torch.float64, device=d); b = torch.randn(n, n, dtype=torch.float64, device=d)
    s = t(lambda: a @ b)
    print(f"dgemm n={n}: {2*n**3/s/1e12:.2f} TF/s")
for n in (4096, 2048, 1024, 512):
    a = torch.randn(n, n, dtype=torch.float64, device=d) + n * torch.eye(n, dtype=torch.float64, device=d)
    s = t(lambda: torch.linalg.lu_factor(a))
    print(f"getrf n={n}: {2/3*n**3/s/1e12:.2f} TF/s ({s*1e3:.2f} ms)")
    s = t(lambda: torch.linalg.inv(a))
    print(f"inv n={n}: {2*n**3/s/1e12:.2f} TF/s (2n^3) ({s*1e3:.2f} ms)")
for n, bt in ((1024, 16), (512, 64), (256, 128)):
    a = torch.randn(bt, n, n, dtype=torch.float64, device=d) + n * torch.eye(n, dtype=torch.float64, device=d)
    s = t(lambda: torch.linalg.inv(a))
    print(f"batched inv n={n} x{bt}: {bt*2*n**3/s/1e12:.2f} TF/s ({s*1e3:.2f} ms)")
