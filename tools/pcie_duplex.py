"""Pinned host <-> device copy bandwidth, one direction at a time and both at
once on two streams (is PCIe full duplex for the pipelined integrate?)."""
import json
import time

import torch


def main():
    n = 1 << 30                                   # 8 GiB of float64 per buffer
    h_src = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h_dst = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d_a = torch.empty(n, dtype=torch.float64, device="cuda")
    d_b = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    gb = n * 8 / 1e9
    out = {}
    for label, h2d, d2h in (("h2d", True, False), ("d2h", False, True), ("both", True, True),
                            ("h2d_2", True, False), ("both_2", True, True)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_src, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_dst.copy_(d_b, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[label] = {"s": round(dt, 4), "GBps_each": round(gb / dt, 1),
                      "GBps_total": round(gb * (h2d + d2h) / dt, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
