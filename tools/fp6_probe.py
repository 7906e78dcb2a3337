"""Probe (one-off): FP6 E3M2 operand container convention of tcgen05 kind::f8f6f4."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2501_02625_b200 import halo


def e3m2_value(c):
    c = np.asarray(c, dtype=np.int64)
    s = np.where(c & 0x20, -1.0, 1.0)
    e = (c >> 2) & 7
    m = c & 3
    v = np.where(e == 0, m * 2.0 ** -4, (1 + m / 4.0) * 2.0 ** (e - 3))
    return s * v


rng = np.random.default_rng(0)
M, N, K = 256, 256, 256
ca = rng.integers(0, 64, size=(M, K))
cb = rng.integers(0, 64, size=(N, K))
ref = e3m2_value(ca) @ e3m2_value(cb).T
one = torch.ones(1, device="cuda")
code = os.environ.get("HALO_GEMM_F6_CODE", "default")
for name, f in (("low6", lambda c: c), ("high6", lambda c: c << 2)):
    for amaj, bmaj in ((True, True), (False, True)):
        A = torch.from_numpy(f(ca).astype(np.uint8)).cuda()
        B = torch.from_numpy(f(cb).astype(np.uint8)).cuda()
        Ad = A if amaj else A.t().contiguous()
        Bd = B if bmaj else B.t().contiguous()
        try:
            C = halo.qmatmul(Ad, Bd, one, one, a_kmajor=amaj, b_kmajor=bmaj, fmt=2).cpu().numpy()
            err = np.abs(C - ref).max() / np.abs(ref).max()
            cc = np.corrcoef(C.ravel(), ref.ravel())[0, 1]
            print("code", code, name, "a_kmajor", amaj, "b_kmajor", bmaj, "max rel err", round(float(err), 4), "corr", round(float(cc), 4), flush=True)
        except Exception as e:
            print(name, amaj, bmaj, "error", e, flush=True)

# sanity: E4M3 through the same harness
ce = rng.integers(0, 256, size=(M, K)); ce = np.where((ce & 0x7f) == 0x7f, 0, ce)
de = rng.integers(0, 256, size=(N, K)); de = np.where((de & 0x7f) == 0x7f, 0, de)
def e4m3_value(c):
    c = np.asarray(c, dtype=np.int64); s = np.where(c & 0x80, -1.0, 1.0); e = (c >> 3) & 15; m = c & 7
    return s * np.where(e == 0, m * 2.0 ** -9, (1 + m / 8.0) * 2.0 ** (e - 7))
refe = e4m3_value(ce) @ e4m3_value(de).T
Ce = halo.qmatmul(torch.from_numpy(ce.astype(np.uint8)).cuda(), torch.from_numpy(de.astype(np.uint8)).cuda(), one, one, fmt=1).cpu().numpy()
print("e4m3 sanity rel err", float(np.abs(Ce - refe).max() / np.abs(refe).max()))
