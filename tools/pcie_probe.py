"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently (GB/s)."""
import json
import torch

def bw(n_bytes, fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return n_bytes * reps / (a.elapsed_time(b) / 1e3) / 1e9

N = 2_830_000_000
hd = torch.empty(N, dtype=torch.uint8, device="cuda")
hh = torch.empty(N, dtype=torch.uint8, pin_memory=True)
small = 407_000_000
sd = torch.empty(small, dtype=torch.uint8, device="cuda")
sh = torch.empty(small, dtype=torch.uint8, pin_memory=True)
out = {}
out["d2h_GBps"] = bw(N, lambda: hh.copy_(hd, non_blocking=True))
out["h2d_GBps"] = bw(N, lambda: hd.copy_(hh, non_blocking=True))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1):
        hh.copy_(hd, non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(7):
            sd.copy_(sh, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
out["d2h_with_concurrent_h2d_GBps"] = bw(N, both)
# two D2H streams in parallel (halves)
h1, h2 = hh[: N // 2], hh[N // 2:]
d1, d2 = hd[: N // 2], hd[N // 2:]
def two():
    with torch.cuda.stream(s1):
        h1.copy_(d1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
out["d2h_two_streams_GBps"] = bw(N, two)
print(json.dumps(out))
