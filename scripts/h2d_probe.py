"""Pinned host -> device copy bandwidth for the e2e leg: one 512 MiB copy vs
the same bytes split over 2 / 4 streams (probe, not product code)."""
import torch

n = 512 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(k):
    cur = torch.cuda.current_stream()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(cur)
    chunk = n // k
    for i in range(k):
        st = streams[i % len(streams)]
        st.wait_event(s)
        with torch.cuda.stream(st):
            d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
    for i in range(min(k, len(streams))):
        cur.wait_stream(streams[i])
    e.record(cur)
    torch.cuda.synchronize()
    return s.elapsed_time(e)


for k in (1, 2, 4, 8, 1, 2, 4):
    run(k)
    t = min(run(k) for _ in range(5))
    print(f"{k} chunk(s): {t:.3f} ms  {n / t / 1e6:.1f} GB/s")
