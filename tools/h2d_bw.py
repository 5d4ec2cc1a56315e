import torch, time
x = torch.empty(402_653_200 // 4, dtype=torch.int32).pin_memory()
y = torch.empty_like(x, device='cuda')
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"H2D 402 MB pinned: {1e3*(t1-t0):.2f} ms = {402.65/(t1-t0)/1e3:.1f} GB/s")
