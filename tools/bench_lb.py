"""Left large-block K2 (fwht_cols_lb.cu) micro-run: left_rotate_quantize
(phase A + phase B) at 8192 tokens, with and without the plain codes; also
the driver for the ncu capture.
  python tools/bench_lb.py [hidden] [block] [reps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402

hidden = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
block = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
e = (torch.randn(8192, hidden, device="cuda") * 1e-3).to(torch.bfloat16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def t(fn):
    ts = []
    for i in range(reps + 2):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


n = e.numel()
for plain in (True, False):
    ms = t(lambda: halo.left_rotate_quantize(e, block, fmt=0, plain=plain))
    print(f"hidden {hidden} block {block} plain {plain}: {ms * 1e3:.1f} us, "
          f"{(4 if plain else 3) * n / ms / 1e6:.0f} GB/s algorithmic")
