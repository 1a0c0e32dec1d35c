"""Pinned host -> device copy bandwidth on this box (the e2e ceiling of config 3):
one stream with chunk sizes 8 MB .. 1 GB, and two / four streams splitting each chunk."""
import torch

torch.cuda.init()
total = 2 << 30
src = torch.empty(total, dtype=torch.uint8).pin_memory()
dst = torch.empty(total, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(chunk, nstreams, reps=3):
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in streams[:nstreams]:
            s.wait_event(e0)
        off, i = 0, 0
        while off < total:
            n = min(chunk, total - off)
            with torch.cuda.stream(streams[i % nstreams]):
                dst[off:off + n].copy_(src[off:off + n], non_blocking=True)
            off += n
            i += 1
        for s in streams[:nstreams]:
            e1.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, total / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


for ns in (1, 2, 4):
    for mb in (8, 32, 128, 512, 1024):
        print(f"streams {ns} chunk {mb:5d} MB: {run(mb << 20, ns):6.1f} GB/s", flush=True)
