"""Host->device (and device->host) copy bandwidth of the e2e step's upload pattern (per view:
dcolor, ddepth, dsemantics, dkmap, dnormals of a 1200x680, C=50 frame; 8
views) from pinned memory: one copy stream vs the views spread over 2 / 4
streams, idle GPU vs a concurrent HBM-heavy kernel.  GPU box only.

    python tools/h2d_probe.py
"""
import time

import torch


def main():
    dev = torch.device("cuda:0")
    W, H, C, V = 1200, 680, 50, 8
    shapes = [(3, H, W), (H, W), (C, H, W), (H, W), (3, H, W)]
    host = [[torch.randn(*s).pin_memory() for s in shapes] for _ in range(V)]
    dst = [[torch.empty(*s, device=dev) for s in shapes] for _ in range(V)]
    nbytes = sum(t.numel() * 4 for v in host for t in v)
    streams = [torch.cuda.Stream(dev) for _ in range(4)]
    busy_a = torch.empty(512 << 20, dtype=torch.float32, device=dev)  # 2 GB
    busy_b = torch.empty_like(busy_a)

    def run(nstreams, busy):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if busy:
            bs = torch.cuda.Stream(dev)
            with torch.cuda.stream(bs):
                for _ in range(20):
                    busy_b.copy_(busy_a)
        for j in range(V):
            with torch.cuda.stream(streams[j % nstreams]):
                for d, h in zip(dst[j], host[j]):
                    d.copy_(h, non_blocking=True)
        for s in streams[:nstreams]:
            s.synchronize()
        dt = time.perf_counter() - t
        torch.cuda.synchronize()
        return nbytes / dt / 1e9

    def run_d2h(nstreams):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for j in range(V):
            with torch.cuda.stream(streams[j % nstreams]):
                for d, h in zip(dst[j], host[j]):
                    h.copy_(d, non_blocking=True)
        for s in streams[:nstreams]:
            s.synchronize()
        return nbytes / (time.perf_counter() - t) / 1e9

    for ns in (1, 2):
        run_d2h(ns)
        r = sorted(run_d2h(ns) for _ in range(5))
        print(f"device->host streams={ns}: {r[2]:.1f} GB/s (median of 5)")
    for busy in (False, True):
        for ns in (1, 2, 4):
            run(ns, busy)
            r = sorted(run(ns, busy) for _ in range(5))
            print(f"streams={ns} concurrent_hbm_copy={busy}: {r[2]:.1f} GB/s (median of 5; {nbytes / 1e9:.2f} GB)")


if __name__ == "__main__":
    main()
