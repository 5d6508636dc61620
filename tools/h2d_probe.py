"""H2D bandwidth from pinned host memory: one copy stream vs two, chunk sizes."""
import time
import torch

n = 12_800_000_000 // 8
H = torch.empty(n, dtype=torch.float64, pin_memory=True)
D = torch.empty(n, dtype=torch.float64, device="cuda")
H.fill_(1.0)
for streams in (1, 2, 4):
    for chunk_mb in (64, 256):
        ch = chunk_mb * (1 << 20) // 8
        ss = [torch.cuda.Stream() for _ in range(streams)]
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i, off in enumerate(range(0, n, ch)):
                with torch.cuda.stream(ss[i % streams]):
                    D[off:off + ch].copy_(H[off:off + ch], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"streams={streams} chunk={chunk_mb}MB: {n * 8 / dt / 1e9:.1f} GB/s", flush=True)
