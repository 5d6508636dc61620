"""Host-feeder throughput: dataset_suffstats from an SSTATBIN file in /dev/shm (page cache),
from pageable numpy memory and from pinned memory, vs feeder thread count.  Prints one JSON
line per case; checks every case gives the same bits.

    python tools/feeder_probe.py [rows] [p]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23826_b200 as s  # noqa: E402


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    eng = s.Engine(0)
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    eng.generate(D, 0, 42, 1.0, 2, 0, n, p)
    pinned = torch.empty((n, p), dtype=torch.float64, pin_memory=True)
    pinned.copy_(D)
    host = pinned.numpy().copy()  # pageable
    del D
    torch.cuda.empty_cache()
    d = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"
    path = os.path.join(d, f"feeder_{os.getpid()}.bin")
    hdr = bytearray(64)
    hdr[0:8] = b"SSTATBIN"
    hdr[8:12] = (1).to_bytes(4, "little")
    hdr[12:20] = n.to_bytes(8, "little")
    hdr[20:24] = p.to_bytes(4, "little")
    with open(path, "wb") as f:
        f.write(hdr)
        host.tofile(f)
    schema = s.DatasetSchema.generic(p, False)
    plan = s.ReductionPlan(s.plan_partitions(n, 1 << 20))
    ref = None
    try:
        cases = [("pinned", pinned, [0])] + [("pageable", host, [1, 4, 8, 16])] + [("file", path, [1, 4, 8, 16])]
        for kind, src, threads in cases:
            for t in threads:
                eng.set_host_threads(t)
                best = None
                for _ in range(3):
                    t0 = time.perf_counter()
                    got = eng.dataset_suffstats(src, schema, plan)
                    dt = time.perf_counter() - t0
                    best = dt if best is None else min(best, dt)
                if ref is None:
                    ref = got
                assert got.bit_equal(ref), (kind, t)
                print(json.dumps({"source": kind, "host_threads": t, "rows": n, "p": p, "s": round(best, 4),
                                  "rows_per_s": n / best, "GB_per_s": n * p * 8 / best / 1e9}), flush=True)
    finally:
        os.remove(path)


if __name__ == "__main__":
    main()
