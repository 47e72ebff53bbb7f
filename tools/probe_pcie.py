"""PCIe floor of the TM-1 e2e step: one step's H2D (13.7 MB) and D2H (23.8 MB) from/to pinned
host memory, each direction alone and both at once on two streams (as gputx_run_bulks overlaps
them), 10 repetitions each, best and median."""
import statistics
import sys

import torch

h2d_b = int(sys.argv[1]) if len(sys.argv) > 1 else 13_678_682
d2h_b = int(sys.argv[2]) if len(sys.argv) > 2 else 23_802_596
dev = torch.device("cuda:0")
hi, di = torch.empty(h2d_b, dtype=torch.uint8).pin_memory(), torch.empty(h2d_b, dtype=torch.uint8, device=dev)
ho, do = torch.empty(d2h_b, dtype=torch.uint8).pin_memory(), torch.empty(d2h_b, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def run(mode, reps=10):
    out = []
    for _ in range(reps + 2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        s1.wait_event(e0)
        s2.wait_event(e0)
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1):
                di.copy_(hi, non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2):
                ho.copy_(do, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
        e1.record(cur)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    out = out[2:]
    return min(out), statistics.median(out)


for m in ("h2d", "d2h", "both", "h2d", "both"):
    b, med = run(m)
    print(f"{m:5s} best {b:.3f} ms median {med:.3f} ms")
