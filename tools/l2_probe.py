"""L2-resident copy bandwidth on one B200: y.copy_(x) repeated over working
sets below and above the 126 MB L2 (read + write bytes / time)."""
import torch
torch.cuda.init()
for mb in (16, 32, 64, 96, 128, 256, 1024):
    n = mb * 2**20 // 8                      # two buffers of mb/2 MB each
    x = torch.randn(n, device="cuda")
    y = torch.empty_like(x)
    for _ in range(20):
        y.copy_(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 200
    e0.record()
    for _ in range(reps):
        y.copy_(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"working set {mb} MB: {2 * n * 4 / (ms * 1e-3) / 1e9:.0f} GB/s ({ms * 1e3:.1f} us per copy)", flush=True)
