"""Fiber statistics of a config: distinct (i_n, i_x) pairs per mode pair (GPU, torch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import sacd_inputs as SI
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = SI.CONFIGS[name]
c, v = SI.make_tensor(cfg, device="cuda")
c = c.long()
nnz = c.shape[0]
d = cfg.dims
print(name, "nnz", nnz, "dims", d)
for x, y in ((0, 1), (0, 2), (1, 2)):
    key = c[:, x] * d[y] + c[:, y]
    n = torch.unique(key).numel()
    print(f"distinct ({x},{y}) pairs: {n}  mean fiber length {nnz / n:.3f}")
for m in range(3):
    cnt = torch.bincount(c[:, m], minlength=d[m])
    top = torch.sort(cnt, descending=True).values
    print(f"mode {m}: max slice {top[0].item()} ({100*top[0].item()/nnz:.2f}%), top-400 rows hold {100*top[:400].sum().item()/nnz:.1f}% , empty rows {(cnt==0).sum().item()}")
