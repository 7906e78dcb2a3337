"""RMSNorm forward / backward at the Llama block shape (8192 x 4096, bf16): the plain and
the residual-gradient (RES) forms through the C ABI, CUDA-event times.
Usage: python tools/bench_norm.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402
from paper_2501_02625_b200._lib import check, lib  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rows, dim = 8192, 4096
bf = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(rows, dim, generator=g, device="cuda").to(bf)
dy = torch.randn(rows, dim, generator=g, device="cuda").to(bf)
dres = torch.randn(rows, dim, generator=g, device="cuda").to(bf)
w = torch.rand(dim, generator=g, device="cuda") + 0.5
a = torch.empty_like(x)
rstd = torch.empty(rows, dtype=torch.float32, device="cuda")
check(lib().halo_rmsnorm_forward(halo._ptr(x), halo._ptr(w), halo._ptr(a), 1, halo._ptr(rstd), rows, dim, 1, 1e-5,
                                 halo._stream()))
dx = torch.empty_like(x)
dw = torch.empty(dim, dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def res():
    check(lib().halo_rmsnorm_backward_res(halo._ptr(x), halo._ptr(dy), 1, halo._ptr(w), halo._ptr(rstd),
                                          halo._ptr(dres), halo._ptr(dx), halo._ptr(dw), rows, dim, halo._stream()))


def plain():
    check(lib().halo_rmsnorm_backward(halo._ptr(x), halo._ptr(dy), 1, halo._ptr(w), halo._ptr(rstd), halo._ptr(dx),
                                      halo._ptr(dw), rows, dim, 1, halo._stream()))


h_ = torch.empty_like(x)


def fwd():
    check(lib().halo_rmsnorm_forward(halo._ptr(x), halo._ptr(w), halo._ptr(a), 1, halo._ptr(rstd), rows, dim, 1, 1e-5,
                                     halo._stream()))


def fwd_add():
    check(lib().halo_add_rmsnorm_forward(halo._ptr(x), halo._ptr(dres), halo._ptr(w), halo._ptr(h_), halo._ptr(a),
                                         halo._ptr(rstd), rows, dim, 1e-5, halo._stream()))


NBYTES = {"res": 4, "plain": 3, "fwd": 2, "fwd_add": 4}
for name, fn in (("res", res), ("plain", plain), ("fwd", fwd), ("fwd_add", fwd_add)):
    for _ in range(3):
        fn()
    t = 0.0
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t += e0.elapsed_time(e1)
    ms = t / reps
    nbytes = rows * dim * 2 * NBYTES[name]
    print(f"{name}: {ms * 1e3:.1f} us  ({nbytes / ms / 1e6:.0f} GB/s over {nbytes / 1e6:.0f} MB)")
