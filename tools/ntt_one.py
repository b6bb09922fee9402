"""One forward + one inverse NTT launch at (log2n, L, batch) for profiling."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2509_01253_b200.ntt import RnsNtt
logn, L, B = (int(a) for a in sys.argv[1:4])
pl = RnsNtt(logn, L, 50, device=0)
P = torch.tensor(pl.primes.view(np.int64), device="cuda")
x = torch.remainder(torch.randint(0, 1 << 62, (B, L, 1 << logn), device="cuda", dtype=torch.int64), P[None, :, None])
for _ in range(2):
    pl.forward(x)
    pl.inverse(x)
torch.cuda.synchronize()
