"""Pinned host -> device copy rate for 1 GiB: one cudaMemcpyAsync vs the same
bytes split into chunks over several streams (copy-engine concurrency)."""
import torch
n = 1 << 28
h = torch.empty(n, dtype=torch.float32).pin_memory()
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for nstream in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nstream)]
    chunk = n // nstream
    best = 1e9
    for rep in range(6):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for i, s in enumerate(streams):
            s.wait_event(a)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{nstream} streams: {best:.2f} ms = {4 * n / best / 1e6:.1f} GB/s")
