#!/usr/bin/env python
"""One Python-API mgpu SYMV and GEMV call (2 logical GPUs on device 0),
for an ncu launch list: every launch must be a library (kblas_) kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1410_1726_b200 as kb  # noqa: E402

n, nb, G = 8192, 128, 2
A = torch.empty(n, n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
dm = kb.distribute(kb.view_of(A.T), nb, G)
x = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
y = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for beta in (0.0, 0.5):
    kb.symv_hemv_mgpu("l", 1.0, dm, x, beta, y, kb.KernelConfig(nb, 2))
    kb.gemv_mgpu("n", 1.0, dm, x, beta, y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
