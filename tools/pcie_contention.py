"""Do concurrent SpMV kernels slow PCIe copies?  H2D+D2H of 134 MB each,
alone and alongside an SpMV loop on a third stream (SPMV_CTAS_PER_SM caps
the kernel's CTAs when set)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2304_09511_b200 as sp  # noqa: E402

n = 256 ** 3
xh = torch.rand(n, dtype=torch.float64).pin_memory()
yh = torch.empty(n, dtype=torch.float64).pin_memory()
xd = torch.empty(n, dtype=torch.float64, device="cuda")
yd = torch.rand(n, dtype=torch.float64, device="cuda")
A = sp.gen_stencil27(256, 256, 256)
xs = torch.rand(n, dtype=torch.float64, device="cuda")
ys = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def copies(with_kernel: bool, reps: int = 5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        if with_kernel:
            with torch.cuda.stream(s3):
                for _ in range(6):
                    sp.spmv_csr_plain(A, xs, out=ys)
        a = torch.cuda.Event(enable_timing=True)
        b1, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s1)
        s2.wait_event(a)
        with torch.cuda.stream(s1):
            xd.copy_(xh, non_blocking=True)
            b1.record(s1)
        with torch.cuda.stream(s2):
            yh.copy_(yd, non_blocking=True)
            b2.record(s2)
        torch.cuda.synchronize()
        ts.append((a.elapsed_time(b1), a.elapsed_time(b2)))
    return sorted(ts)[len(ts) // 2]


sp.spmv_csr_plain(A, xs, out=ys)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    sp.spmv_csr_plain(A, xs, out=ys)
torch.cuda.synchronize()
print("spmv %.3f ms" % ((time.perf_counter() - t0) / 10 * 1e3))
print("copies alone   H2D %.3f D2H %.3f ms" % copies(False))
print("copies + spmv  H2D %.3f D2H %.3f ms" % copies(True))


def chunked(nchunks: int, reps: int = 5):
    ts = []
    step = n // nchunks
    for _ in range(reps):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b1, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s1)
        s2.wait_event(a)
        for c in range(nchunks):
            lo, hi = c * step, (c + 1) * step if c < nchunks - 1 else n
            with torch.cuda.stream(s1):
                xd[lo:hi].copy_(xh[lo:hi], non_blocking=True)
            with torch.cuda.stream(s2):
                yh[lo:hi].copy_(yd[lo:hi], non_blocking=True)
        b1.record(s1)
        b2.record(s2)
        torch.cuda.synchronize()
        ts.append((a.elapsed_time(b1), a.elapsed_time(b2)))
    return sorted(ts)[len(ts) // 2]


for nc in (1, 4, 16, 48):
    print("chunked %2d      H2D %.3f D2H %.3f ms" % ((nc,) + chunked(nc)))


def gated(nchunks: int, kernel: bool, reps: int = 5):
    """The pipeline's dependency pattern: all H2D chunks first on s1; D2H
    chunk c on s2 waits for H2D chunk c+1 (and a kernel on s3 if asked)."""
    ts = []
    step = n // nchunks
    for _ in range(reps):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b2 = torch.cuda.Event(enable_timing=True)
        a.record(s1)
        s2.wait_event(a)
        s3.wait_event(a)
        evs = []
        for c in range(nchunks):
            lo, hi = c * step, (c + 1) * step if c < nchunks - 1 else n
            with torch.cuda.stream(s1):
                xd[lo:hi].copy_(xh[lo:hi], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s1)
                evs.append(e)
        for c in range(nchunks):
            lo, hi = c * step, (c + 1) * step if c < nchunks - 1 else n
            gate = evs[min(c + 1, nchunks - 1)]
            if kernel:
                s3.wait_event(gate)
                with torch.cuda.stream(s3):
                    yd[lo:hi].mul_(1.0)
                    g2 = torch.cuda.Event()
                    g2.record(s3)
                s2.wait_event(g2)
            else:
                s2.wait_event(gate)
            with torch.cuda.stream(s2):
                yh[lo:hi].copy_(yd[lo:hi], non_blocking=True)
        b2.record(s2)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b2))
    return sorted(ts)[len(ts) // 2]


for nc in (8, 24):
    print("gated %2d: no kernel %.3f ms, with kernel %.3f ms" % (nc, gated(nc, False), gated(nc, True)))
