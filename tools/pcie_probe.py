"""PCIe probe: pinned H2D alone, D2H alone, and both directions at once on two streams (GB/s).

Decides whether the end-to-end bench can overlap its input uploads with its result downloads.
"""
import torch


def main():
    n = 512 << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        cur = torch.cuda.current_stream()
        cur.wait_stream(s1)
        cur.wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e-3

    def h2d():
        with torch.cuda.stream(s1):
            s1.wait_stream(torch.cuda.current_stream())
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            s2.wait_stream(torch.cuda.current_stream())
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(f"H2D {n / t1 / 1e9:.1f} GB/s, D2H {n / t2 / 1e9:.1f} GB/s, "
          f"both at once {2 * n / t3 / 1e9:.1f} GB/s aggregate ({t3 * 1e3:.2f} ms vs {(t1 + t2) * 1e3:.2f} serial)")


if __name__ == "__main__":
    main()
