"""D2H / H2D bandwidth of pinned host memory on this box: one copy vs several streams vs
chunks (the e2e path's 8.6 GB solution read-back)."""
import json
import sys
import time

import torch

n = int(float(sys.argv[1]) if len(sys.argv) > 1 else 8.58e9) // 8
dev = torch.device("cuda:0")
d = torch.empty(n, dtype=torch.float64, device=dev)
h = torch.empty(n, dtype=torch.float64).pin_memory()
res = {}


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for name, ns, nchunk in (("one_copy", 1, 1), ("2_streams", 2, 2), ("4_streams", 4, 4), ("chunks_64_1s", 1, 64),
                         ("chunks_64_4s", 4, 64)):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    size = (n + nchunk - 1) // nchunk

    def run():
        for c in range(nchunk):
            s = streams[c % ns]
            with torch.cuda.stream(s):
                h[c * size:(c + 1) * size].copy_(d[c * size:(c + 1) * size], non_blocking=True)
        for s in streams:
            s.synchronize()

    run()
    t = min(timed(run) for _ in range(3))
    res["d2h_" + name] = 8 * n / t / 1e9
t = min(timed(lambda: d.copy_(h, non_blocking=True)) for _ in range(3))
res["h2d_one_copy"] = 8 * n / t / 1e9
print(json.dumps(res))
