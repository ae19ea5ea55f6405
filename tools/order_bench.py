"""K5 timing (development tool): pdg_order on n packed keys, begin_bit 32,
CUDA events, mean of reps (the event clock ticks in 2.048 us), L2 flushed
between launches.  Run with
PDG_LIB_PATH pointing at another build to compare implementations.
Usage: python tools/order_bench.py [n ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_14851_b200 import _lib  # noqa: E402


def bench(n, reps=30):
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(n)
    hi = (torch.rand(n, device=dev, generator=g) * 100).view(torch.int32).to(torch.int64)
    k = (hi << 32) | torch.arange(n, device=dev, dtype=torch.int64)
    s = torch.arange(n, device=dev, dtype=torch.int32)
    ko, so = torch.empty_like(k), torch.empty_like(s)
    temp = torch.empty(max(int(L.pdg_order_temp_bytes(n)), 16), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def run():
        _lib.check(L.pdg_order(_lib.ptr(k), _lib.ptr(ko), _lib.ptr(s), _lib.ptr(so), n, 32,
                               _lib.ptr(temp), temp.numel(), _lib.stream_ptr()), "pdg_order")
    for _ in range(3):
        run()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda._sleep(200_000)              # stream busy while the host launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ok = bool(torch.all(ko[1:] >= ko[:-1]).item())
    return {"n": n, "ms": float(np.mean(ts)), "sorted": ok}


if __name__ == "__main__":
    ns = [int(x) for x in sys.argv[1:]] or [100_000, 1_000_000]
    print(json.dumps({"lib": os.environ.get("PDG_LIB_PATH", "in-tree"),
                      "runs": [bench(n) for n in ns]}))
