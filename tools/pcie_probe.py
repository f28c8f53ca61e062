"""PCIe bandwidth of the e2e arm's transfers: pinned H2D alone, D2H alone, and both at once (full duplex),
with the bench's per-step byte counts (1.258 GB in, 1.057 GB out)."""
import torch

dev = torch.device("cuda", 0)
n_in, n_out = 1258291200, 1056964608
hi = torch.empty(n_in, dtype=torch.uint8, pin_memory=True)
ho = torch.empty(n_out, dtype=torch.uint8, pin_memory=True)
di = torch.empty(n_in, dtype=torch.uint8, device=dev)
do = torch.empty(n_out, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(f, reps=5):
    f()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(reps):
        f()
    en.record()
    torch.cuda.synchronize()
    return st.elapsed_time(en) / reps


def h2d():
    di.copy_(hi, non_blocking=True)


def d2h():
    ho.copy_(do, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D alone {n_in / t1 / 1e6:.1f} GB/s ({t1:.2f} ms); D2H alone {n_out / t2 / 1e6:.1f} GB/s ({t2:.2f} ms); "
      f"both at once {t3:.2f} ms (H2D-bound floor of the e2e step)")
for mb in (8, 32, 134):
    n = mb * 1 << 20
    t = timed(lambda: di[:n].copy_(hi[:n], non_blocking=True), reps=20)
    print(f"H2D chunk {mb} MiB: {n / t / 1e6:.1f} GB/s")
