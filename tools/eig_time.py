"""Development aid: time the full symmetric eigendecomposition (cuSOLVER via torch) at solver sizes."""
import sys
import time

import torch

for n in [int(x) for x in sys.argv[1].split(",")]:
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    A = A + A.T
    torch.linalg.eigh(A)
    torch.cuda.synchronize()
    t = time.time()
    w, V = torch.linalg.eigh(A)
    torch.cuda.synchronize()
    t1 = time.time() - t
    t = time.time()
    w = torch.linalg.eigvalsh(A)
    torch.cuda.synchronize()
    print(f"n={n} eigh {t1:.3f}s eigvalsh {time.time() - t:.3f}s", flush=True)
