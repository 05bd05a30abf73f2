"""Host<->device copy throughput for the e2e operand sizes (pinned host
buffers, CUDA events): H2D alone, D2H alone, both directions concurrently on
two streams.  python tools/pcie_probe.py [MB ...]"""
import sys

import torch


def main():
    sizes = [float(a) for a in sys.argv[1:]] or [0.0625, 1.0, 4.0, 64.0]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for mb in sizes:
        n = int(mb * (1 << 20)) // 16
        h_in = torch.empty(n, dtype=torch.complex128).pin_memory()
        h_out = torch.empty(n, dtype=torch.complex128).pin_memory()
        d_in = torch.empty(n, dtype=torch.complex128, device="cuda")
        d_out = torch.empty(n, dtype=torch.complex128, device="cuda")
        reps = max(10, int(200 / max(mb, 0.1)))

        def timed(fn):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps * 1e-3

        def h2d():
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)

        def d2h():
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)

        def both():
            h2d()
            d2h()

        torch.cuda.current_stream().wait_stream(s1)
        for name, fn in (("H2D", h2d), ("D2H", d2h), ("both", both)):
            t = timed(fn)
            gbs = (2 if name == "both" else 1) * n * 16 / t / 1e9
            print(f"{mb:8.4f} MB {name:5s}: {t * 1e6:8.1f} us per copy (set), {gbs:6.1f} GB/s")


if __name__ == "__main__":
    main()
