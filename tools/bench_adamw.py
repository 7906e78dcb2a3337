"""halo_adamw_step at the cfg5 shard sizes (bf16 master, fp32 grad, fp32 m/v:
24 B/param), CUDA-event times and bandwidth.  Usage: python tools/bench_adamw.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402
from paper_2501_02625_b200._lib import check, lib  # noqa: E402

for n in (4096 * 4096, 6144 * 4096, 14336 * 4096):
    p = torch.randn(n, device="cuda").to(torch.bfloat16)
    g = torch.randn(n, device="cuda") * 1e-3
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")

    def step():
        check(lib().halo_adamw_step(halo._ptr(p), 1, halo._ptr(g), 0, halo._ptr(m), halo._ptr(v), n, 1e-4, 0.9, 0.95,
                                    1e-8, 0.01, 0.1, 0.05, halo._stream()))
    for _ in range(3):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        step()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    print(f"n={n / 1e6:.1f}M: {us:.1f} us, {24 * n / us / 1e3:.0f} GB/s")
