"""Investigation: host->device copy rate of a 2.15 GB pinned buffer with 1, 2 or 4 concurrent streams."""
import torch

n = 2147680256 // 4
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for parts in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    chunk = (n + parts - 1) // parts
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"{parts} stream(s): {ms:.2f} ms = {n * 4 / ms / 1e6:.1f} GB/s", flush=True)
