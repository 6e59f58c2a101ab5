"""fp64 rates of the library's own DMMA GEMM (pmns_dgemm) and dense inverse on this GPU.  Diagnostic only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2510_22077_b200 import _lib  # noqa: E402


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


for n in (8192, 4096, 2048, 1024, 512):
    a = torch.randn(1, n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(1, n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for tr in (False, True):
        s = t(lambda: _lib.dgemm(a, b, c, transA=tr))
        print(f"pmns_dgemm n={n} transA={int(tr)}: {2 * n ** 3 / s / 1e12:.2f} TF/s", flush=True)
    s = t(lambda: a[0] @ b[0])
    print(f"cublas dgemm n={n}: {2 * n ** 3 / s / 1e12:.2f} TF/s", flush=True)
for (m, n, k) in ((2048, 2048, 256), (4096, 4096, 64), (512, 8192, 512), (256, 256, 4096)):
    a = torch.randn(1, k, m, dtype=torch.float64, device="cuda")
    b = torch.randn(1, n, k, dtype=torch.float64, device="cuda")
    c = torch.empty(1, n, m, dtype=torch.float64, device="cuda")
    s = t(lambda: _lib.dgemm(a, b, c))
    print(f"pmns_dgemm m={m} n={n} k={k}: {2 * m * n * k / s / 1e12:.2f} TF/s", flush=True)
for (bt, n) in ((64, 256), (16, 1024)):
    a = torch.randn(bt, n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(bt, n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    s = t(lambda: _lib.dgemm(a, b, c))
    print(f"pmns_dgemm batch={bt} n={n}: {bt * 2 * n ** 3 / s / 1e12:.2f} TF/s", flush=True)
