"""Host-side cost of reading 773 MB of factors: pageable numpy vs pinned torch buffers."""
import time
import numpy as np
import torch
n = 773_000_000 // 8
src = torch.empty(n, dtype=torch.float64, device="cuda")
src.fill_(1.0)
torch.cuda.synchronize()
for rep in range(2):
    t = time.perf_counter(); a = np.empty(n); a_t = torch.from_numpy(a); a_t.copy_(src); t1 = time.perf_counter()
    t2 = time.perf_counter(); p = torch.empty(n, dtype=torch.float64, pin_memory=True); t3 = time.perf_counter()
    p.copy_(src); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"pageable np.empty + D2H {1e3*(t1-t):.1f} ms | pinned alloc {1e3*(t3-t2):.1f} ms + D2H {1e3*(t4-t3):.1f} ms")
