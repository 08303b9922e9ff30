import torch, time
x = torch.empty(400_000_000, dtype=torch.int32).pin_memory()
y = torch.empty_like(x, device='cuda')
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print(f"torch pinned H2D {x.numel()*4/1e9:.2f} GB: {x.numel()*4/dt/1e9:.1f} GB/s")
