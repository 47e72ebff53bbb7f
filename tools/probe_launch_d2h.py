"""Diagnostics: does a concurrent large D2H copy slow kernel launches / short kernels on another stream?"""
import torch

dev = torch.device("cuda")
x = torch.zeros(1024, device=dev)
big = torch.empty(41 << 20, dtype=torch.uint8, device=dev)
host = torch.empty(41 << 20, dtype=torch.uint8).pin_memory()
mid = torch.zeros(8 << 20, device=dev)
cs = torch.cuda.Stream()
s = torch.cuda.current_stream()


def run(kind, with_copy, reps=200):
    torch.cuda.synchronize()
    if with_copy:
        with torch.cuda.stream(cs):
            for _ in range(6):
                host.copy_(big, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        if kind == "tiny":
            x.add_(1)
        else:
            mid.add_(1)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for kind in ["tiny", "mid"]:
    for wc in [False, True, False, True]:
        print(kind, "with D2H" if wc else "alone  ", "%.2f us/kernel" % run(kind, wc))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(200):
        x.add_(1)
for wc in [False, True]:
    torch.cuda.synchronize()
    if wc:
        with torch.cuda.stream(cs):
            for _ in range(6):
                host.copy_(big, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    print("graph tiny", "with D2H" if wc else "alone  ", "%.2f us/kernel" % (e0.elapsed_time(e1) / 200 * 1e3))
