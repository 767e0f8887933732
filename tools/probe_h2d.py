"""Pinned host->device bandwidth with 1..4 concurrent streams (e2e ceiling)."""
import torch

n = 64 * 1024 * 1024 // 8
for nstreams in (1, 2, 4):
    for chunks in (1, 4):
        hs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
        ds = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4)]
        ss = [torch.cuda.Stream() for _ in range(nstreams)]
        for it in range(2):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for st in ss:
                st.wait_event(e0)
            reps = 8
            for r in range(reps):
                st = ss[r % nstreams]
                with torch.cuda.stream(st):
                    h, d = hs[r % 4], ds[r % 4]
                    step = n // chunks
                    for c in range(chunks):
                        d[c * step:(c + 1) * step].copy_(h[c * step:(c + 1) * step], non_blocking=True)
            for st in ss:
                e = torch.cuda.Event()
                e.record(st)
                torch.cuda.current_stream().wait_event(e)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"streams {nstreams} chunks {chunks}: {reps * n * 8 / ms / 1e6:.1f} GB/s")
# D2H concurrently with H2D
h = torch.empty(n, dtype=torch.float64).pin_memory(); d = torch.empty(n, dtype=torch.float64, device="cuda")
h2 = torch.empty(n // 10, dtype=torch.float64).pin_memory(); d2 = torch.empty(n // 10, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); s1.wait_event(e0); s2.wait_event(e0)
for r in range(8):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
for st in (s1, s2):
    e = torch.cuda.Event(); e.record(st); torch.cuda.current_stream().wait_event(e)
e1.record(); torch.cuda.synchronize()
print(f"H2D with concurrent D2H: {8 * n * 8 / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
