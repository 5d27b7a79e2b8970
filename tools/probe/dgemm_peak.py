import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2): c = a @ b
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    s.record(); c = a @ b; e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
print("cuBLAS DGEMM 8192^3: %.2f TF/s (best %.2f ms)" % (2 * 8192**3 / best / 1e9, best))
x = torch.empty(2**30 // 8 * 4, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(2): y.copy_(x)
torch.cuda.synchronize(); best = 1e9
for _ in range(5):
    s.record(); y.copy_(x); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
print("copy 4GiB: %.1f GB/s" % (2 * x.numel() * 8 / best / 1e6))
