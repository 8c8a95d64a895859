"""Raw pinned host->device copy bandwidth on the box (the e2e roofline):
3.2 GB pinned buffer copied whole and in 128 / 64 MiB chunks, CUDA events."""
import torch, time
n = 3_200_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunk in (n, 128 << 20, 64 << 20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(3):
        for o in range(0, n, chunk):
            d[o:o+chunk].copy_(h[o:o+chunk], non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print("chunk", chunk, "GB/s", 3 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
