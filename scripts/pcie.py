"""PCIe reference points for the e2e (host-buffer) path: pinned H2D / D2H
alone and concurrently on two streams, at the 8B step's sizes."""

import json

import torch


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = 2048 * 4096
    h_in = [torch.randn(n).to(torch.bfloat16).pin_memory() for _ in range(2)]
    h_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    d_in = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    d_out = torch.randn(n, device="cuda").to(torch.bfloat16)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def h2d():
        for d, h in zip(d_in, h_in):
            d.copy_(h, non_blocking=True)

    def d2h():
        h_out.copy_(d_out, non_blocking=True)

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            h2d()
        with torch.cuda.stream(s2):
            d2h()
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    r = {}
    ms = timed(h2d)
    r["h2d_33.5MB"] = {"ms": round(ms, 4), "GBps": round(4 * n / ms / 1e6, 1)}
    ms = timed(d2h)
    r["d2h_16.8MB"] = {"ms": round(ms, 4), "GBps": round(2 * n / ms / 1e6, 1)}
    ms = timed(both)
    r["concurrent"] = {"ms": round(ms, 4), "GBps_total": round(6 * n / ms / 1e6, 1)}
    print(json.dumps(r))


if __name__ == "__main__":
    main()
