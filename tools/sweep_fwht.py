"""BASELINE.json configs[3]: Hadamard+quantize bandwidth sweep, hidden
2048-16384 x block 32-16384, right-hand (K1, rows of X/W) and left-hand (K2,
token axis of E) sides, INT8 per-tensor, 8192 rows / tokens, bf16 input.
Each op = phase A (absmax) + phase B (quantize) as the layer runs them;
GB/s counts the algorithmic bytes of the op (input once + codes; K2: both
code sets), and the per-pass rates use each pass's own bytes.  L2 flushed
before every timed op; CUDA events; median of 10.

  python tools/sweep_fwht.py > profiles/r01_sweep_fwht.jsonl
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = peaks["hbm_gbs"]


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


rows = 8192
sides = set(sys.argv[1:]) or {"right", "left"}
g = torch.Generator(device=dev).manual_seed(0)
for hidden in ((2048, 4096, 8192, 16384) if "right" in sides else ()):
    x = torch.randn(rows, hidden, generator=g, device=dev).to(torch.bfloat16)
    n = rows * hidden
    for block in (32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384):
        if block > hidden:
            continue
        rec = {"side": "right (K1)", "rows": rows, "hidden": hidden, "block": block}
        try:
            t_a = timeit(lambda: halo.rotate_absmax(x, block))
            t_op = timeit(lambda: halo.rotate_quantize(x, block, fmt=0))
            rec.update({"ms_op": round(t_op, 4), "GBps_op": round(3 * n / t_op / 1e6, 1),
                        "frac_op": round(3 * n / t_op / 1e6 / hbm, 3),
                        "GBps_phaseA": round(2 * n / t_a / 1e6, 1),
                        "GBps_phaseB": round(3 * n / max(t_op - t_a, 1e-6) / 1e6, 1)})
        except Exception as exc:  # noqa: BLE001
            rec["error"] = str(exc)[:120]
        print(json.dumps(rec), flush=True)
    del x
for hidden in ((2048, 4096, 8192, 16384) if "left" in sides else ()):
    e = (torch.randn(rows, hidden, generator=g, device=dev) * 1e-3).to(torch.bfloat16)
    n = rows * hidden
    for block in (32, 64, 128, 256, 512, 1024, 2048, 4096, 8192):
        rec = {"side": "left (K2)", "tokens": rows, "hidden": hidden, "block": block}
        try:
            t_op = timeit(lambda: halo.left_rotate_quantize(e, block, fmt=0))
            rec.update({"ms_op": round(t_op, 4), "GBps_op": round(4 * n / t_op / 1e6, 1),
                        "frac_op": round(4 * n / t_op / 1e6 / hbm, 3)})
        except Exception as exc:  # noqa: BLE001
            rec["error"] = str(exc)[:120]
        print(json.dumps(rec), flush=True)
    del e
