"""Host <-> device copy rates on the GPU box (pinned memory): H2D alone,
D2H alone, and both at once on two streams; the ceiling of bench.py's e2e
(which moves A in and C'^T out every step).  Diagnostic only."""
import torch


def main():
    n = 37_748_736 // 2  # the BERT step's A (fp16 elements)
    h_in = torch.empty(n, dtype=torch.float16).pin_memory()
    h_out = torch.empty(n, dtype=torch.float16).pin_memory()
    d_in = torch.empty(n, dtype=torch.float16, device="cuda")
    d_out = torch.empty(n, dtype=torch.float16, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        d_in.copy_(h_in, non_blocking=True)
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()

    def timed(fn, reps=10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        for _ in range(reps):
            fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    gb = n * 2 / 1e9
    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(f"H2D {gb / t1 * 1e3:.1f} GB/s ({t1:.3f} ms) | D2H {gb / t2 * 1e3:.1f} GB/s ({t2:.3f} ms) | "
          f"both {t3:.3f} ms ({2 * gb / t3 * 1e3:.1f} GB/s total)")


if __name__ == "__main__":
    main()
