"""Diagnostic (not a test): one 86.7 MB pinned H2D copy vs the same bytes as
2 / 4 concurrent copies on separate streams (separate copy engines)."""
import time

import torch


def main():
    n = 169343 * 128
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for parts in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(parts)]
        step = (n + parts - 1) // parts
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(10):
                for i, st in enumerate(streams):
                    with torch.cuda.stream(st):
                        d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, (time.perf_counter() - t0) / 10)
        print(f"{parts} stream(s): {n * 4 / best / 1e9:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
