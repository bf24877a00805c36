"""Host<->device copy bandwidth on this box (bounds the e2e leg of bench.py).

    python tools/pcie_probe.py [--mib 1024]

Measures pinned H2D / D2H with one copy, with the copy split over 2 and 4
streams, H2D and D2H at the same time, and a zero-copy kernel read of mapped
pinned memory (torch's own copy kernel on a host-mapped view is not used: a
plain .cuda() of a pinned tensor is a DMA).  CUDA events, best of 5.
"""

from __future__ import annotations

import argparse
import json

import torch


def timed(fn, reps=5):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    a = ap.parse_args()
    nb = a.mib << 20
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h.random_(0, 255)
    h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
    cur = torch.cuda.current_stream()
    res = {}

    res["h2d_1"] = nb / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9
    res["d2h_1"] = nb / timed(lambda: h2.copy_(d, non_blocking=True)) / 1e9

    for ns in (2, 4, 8):
        streams = [torch.cuda.Stream() for _ in range(ns)]

        def split(dst, src):
            ev = torch.cuda.Event()
            ev.record(cur)
            ch = nb // ns
            for i, s in enumerate(streams):
                s.wait_event(ev)
                with torch.cuda.stream(s):
                    dst[i * ch:(i + 1) * ch].copy_(src[i * ch:(i + 1) * ch], non_blocking=True)
            for s in streams:
                cur.wait_stream(s)
        res[f"h2d_{ns}streams"] = nb / timed(lambda: split(d, h)) / 1e9

    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        ev = torch.cuda.Event()
        ev.record(cur)
        s1.wait_event(ev)
        s2.wait_event(ev)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    t = timed(both)
    res["bidir_total"] = 2 * nb / t / 1e9
    # chunked H2D in 64 MiB pieces on one stream (pipelined serving granularity)
    ch = 64 << 20

    def chunked():
        for i in range(0, nb, ch):
            d[i:i + ch].copy_(h[i:i + ch], non_blocking=True)
    res["h2d_chunked_64MiB"] = nb / timed(chunked) / 1e9

    # zero-copy: our row-gather kernel reading the pinned (UVA-mapped) host buffer
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2503_04398_b200 import _native as N
    lib = N.lib()
    row = 8192
    rows = nb // row
    idx = torch.arange(rows, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")

    def zc(src):
        N.check(lib.smoe_gather_rows(src.data_ptr(), rows, 2, row // 2, idx.data_ptr(), rows, 1,
                                     0, d.data_ptr(), err.data_ptr(), N.stream_ptr()), "gather")
    res["h2d_zero_copy_kernel"] = nb / timed(lambda: zc(h)) / 1e9
    res["d2d_gather_kernel"] = 2 * nb / timed(lambda: zc(d2)) / 1e9
    # DMA engine and a zero-copy kernel sharing one H2D transfer (half each,
    # concurrently): does the link carry more than either alone?
    half = nb // 2
    rows_h = half // row
    idx_h = torch.arange(rows_h, dtype=torch.int64, device="cuda")
    s_dma = torch.cuda.Stream()

    def split_dma_kernel():
        ev = torch.cuda.Event()
        ev.record(cur)
        s_dma.wait_event(ev)
        with torch.cuda.stream(s_dma):
            d[:half].copy_(h[:half], non_blocking=True)
        N.check(lib.smoe_gather_rows(h[half:].data_ptr(), rows_h, 2, row // 2, idx_h.data_ptr(),
                                     rows_h, 1, 0, d[half:].data_ptr(), err.data_ptr(),
                                     N.stream_ptr()), "gather")
        cur.wait_stream(s_dma)
    res["h2d_dma_plus_zero_copy"] = nb / timed(split_dma_kernel) / 1e9
    res["bytes"] = nb
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}))


if __name__ == "__main__":
    main()
