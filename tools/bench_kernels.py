"""Kernel microbenchmarks (cfg2 shapes): K1 rotate+quantize (phase A + B),
K2 left rotate+quantize, K4 transforms, K3 GEMMs.  CUDA events on the
launching stream, L2 flushed (512 MiB write) before every timed launch,
median of N.  Prints one JSON line per op.

  python tools/bench_kernels.py [k1 k2 k4 gemm] [--reps 10]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402

reps = 10
args = [a for a in sys.argv[1:]]
if "--reps" in args:
    i = args.index("--reps")
    reps = int(args[i + 1])
    del args[i:i + 2]
what = set(args or ["k1", "k2", "k4", "gemm"])
dev = torch.device("cuda", 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json"))) if os.path.exists("MEASURED_PEAKS.json") else {}
hbm = peaks.get("hbm_gbs", 6650.0)


def timeit(fn, nbytes=None, ops=None, name="", warm=3, **extra):
    for _ in range(warm):
        fn()
    ts = []
    st = torch.cuda.current_stream()
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    rec = {"op": name, "ms": round(ms, 4), **extra}
    if nbytes:
        rec["GBps"] = round(nbytes / ms / 1e6, 1)
        rec["frac_hbm"] = round(nbytes / ms / 1e6 / hbm, 3)
    if ops:
        rec["TOPS"] = round(ops / ms / 1e9, 1)
    print(json.dumps(rec), flush=True)
    return ms


g = torch.Generator(device=dev).manual_seed(0)
bf = torch.bfloat16
B = 256
shapes = {"X": (8192, 4096), "W_gate": (14336, 4096), "W_down": (4096, 14336), "H": (8192, 14336)}
if "k1" in what:
    for nm, (r, c) in shapes.items():
        a = torch.randn(r, c, generator=g, device=dev).to(bf)
        n = r * c
        timeit(lambda: halo.rotate_absmax(a, B), nbytes=2 * n, name=f"k1_absmax[{nm} {r}x{c}]")
        timeit(lambda: halo.rotate_quantize(a, B), nbytes=3 * n, name=f"k1_quant_AB[{nm} {r}x{c}]",
               note="bytes counted: one bf16 read + int8 write (algorithmic)")
        del a
if "k2" in what:
    for nm, (r, c) in {"dY": (8192, 4096), "dG": (8192, 14336)}.items():
        e = (torch.randn(r, c, generator=g, device=dev) * 1e-3).to(bf)
        n = r * c
        timeit(lambda: halo.left_rotate_quantize(e, B), nbytes=4 * n, name=f"k2_left_quant_AB[{nm} {r}x{c}]")
        del e
if "k4" in what:
    for nm, (r, c) in {"dX_gate": (8192, 4096), "dX_down": (8192, 14336), "dW": (14336, 4096)}.items():
        p = torch.randn(r, c, generator=g, device=dev)
        n = r * c
        timeit(lambda: halo.transform_right(p, B, out_dtype=bf), nbytes=6 * n, name=f"k4_right_bf16[{nm} {r}x{c}]")
        timeit(lambda: halo.transform_left(p, B), nbytes=8 * n, name=f"k4_left_f32[{nm} {r}x{c}]")
        del p
if "gemm" in what:
    b, H, I = 8192, 4096, 14336
    one = torch.ones(1, device=dev)
    xq = torch.randint(-127, 128, (b, H), dtype=torch.int8, device=dev, generator=g)
    wq = torch.randint(-127, 128, (I, H), dtype=torch.int8, device=dev, generator=g)
    eq = torch.randint(-127, 128, (b, I), dtype=torch.int8, device=dev, generator=g)
    timeit(lambda: halo.qmatmul(xq, wq, one, one, out="bf16"), ops=2 * b * H * I, name="gemm_F[8192x14336x4096 NT bf16]")
    timeit(lambda: halo.qmatmul(eq, wq, one, one, b_kmajor=False, out="f32"), ops=2 * b * H * I,
           name="gemm_E[8192x4096x14336 K/MN f32]")
    timeit(lambda: halo.qmatmul(eq, xq, one, one, a_kmajor=False, b_kmajor=False, out="f32"), ops=2 * b * H * I,
           name="gemm_G[14336x4096x8192 MN/MN f32]")
if "gemm_sweep" in what:
    one = torch.ones(1, device=dev)
    def cod(r, c):
        return torch.randint(-127, 128, (r, c), dtype=torch.int8, device=dev, generator=g)
    for (M, N, K, ak, bk, out) in [(8192, 14336, 4096, 1, 1, "bf16"), (8192, 14336, 4096, 1, 1, "f32"),
                                   (8192, 14336, 4096, 1, 1, "s32"), (8192, 4096, 14336, 1, 1, "bf16"),
                                   (8192, 14336, 8192, 1, 1, "bf16"), (16384, 16384, 4096, 1, 1, "bf16"),
                                   (8192, 8192, 8192, 1, 1, "bf16"), (8192, 4096, 14336, 1, 0, "f32"),
                                   (14336, 4096, 8192, 0, 0, "f32")]:
        a = cod(M, K) if ak else cod(K, M)
        b = cod(N, K) if bk else cod(K, N)
        timeit(lambda: halo.qmatmul(a, b, one, one, a_kmajor=bool(ak), b_kmajor=bool(bk), out=out), ops=2 * M * N * K,
               name=f"gemm[{M}x{N}x{K} a{'K' if ak else 'MN'} b{'K' if bk else 'MN'} {out}]")
        del a, b
if "gemm_k" in what:  # per-tile overhead: fixed M x N, growing K
    one = torch.ones(1, device=dev)
    def cod(r, c):
        return torch.randint(-127, 128, (r, c), dtype=torch.int8, device=dev, generator=g)
    for K in (1024, 2048, 4096, 8192, 16384):
        for (M, N, out) in [(8192, 14336, "bf16"), (8192, 14336, "f32")]:
            a, b = cod(M, K), cod(N, K)
            timeit(lambda: halo.qmatmul(a, b, one, one, out=out), ops=2 * M * N * K, name=f"gemm_k[{M}x{N}x{K} {out}]",
                   tiles=(M // 256) * (N // 256))
            del a, b
if "gemm_edown" in what:  # the E GEMM of down_proj (prod^T: M = 14336, N = 8192 tokens, K = 4096)
    one = torch.ones(1, device=dev)
    def cod(r, c):
        return torch.randint(-127, 128, (r, c), dtype=torch.int8, device=dev, generator=g)
    M, N, K = 14336, 8192, 4096
    a, b = cod(K, M), cod(N, K)
    for hb, tr in ((None, False), (256, False), (None, True), (256, True)):
        kw = {} if hb is None else {"had_block": hb}
        timeit(lambda: halo.qmatmul(a, b, one, one, a_kmajor=False, b_kmajor=True, out="f32", transposed=tr, **kw),
               ops=2 * M * N * K, name=f"gemm_edown[aMN bK f32 xf={hb} trans={tr}]")
    a2 = cod(M, K)
    timeit(lambda: halo.qmatmul(a2, b, one, one, out="f32", had_block=256, transposed=True), ops=2 * M * N * K,
           name="gemm_edown[aK bK f32 xf=256 trans=True]")
    del a, b, a2
    for (M, N) in ((14336, 4096), (4096, 14336)):  # the G GEMMs (dW, right transform along N)
        a, b = cod(8192, M), cod(8192, N)
        for hb in (None, 256):
            kw = {} if hb is None else {"had_block": hb}
            timeit(lambda: halo.qmatmul(a, b, one, one, a_kmajor=False, b_kmajor=False, out="f32", **kw),
                   ops=2 * M * N * 8192, name=f"gemm_G[{M}x{N}x8192 aMN bMN f32 xf={hb}]")
        del a, b
if "gemm_epi" in what:
    one = torch.ones(1, device=dev)
    def cod(r, c):
        return torch.randint(-127, 128, (r, c), dtype=torch.int8, device=dev, generator=g)
    for (M, N, K, out) in [(8192, 14336, 128, "bf16"), (8192, 14336, 128, "f32"), (8192, 14336, 128, "s32"),
                           (8192, 14336, 512, "bf16")]:
        a, b = cod(M, K), cod(N, K)
        ms = timeit(lambda: halo.qmatmul(a, b, one, one, out=out), ops=2 * M * N * K, name=f"gemm_epi[{M}x{N}x{K} {out}]",
                    tiles=(M // 256) * (N // 256))
        del a, b
if "fp8" in what:
    for nm, (r, c) in {"dY": (8192, 4096), "dG": (8192, 14336)}.items():
        e = (torch.randn(r, c, generator=g, device=dev) * 1e-3).to(bf)
        n = r * c
        for fmt in (0, 1, 2):
            timeit(lambda: halo.left_rotate_quantize(e, B, fmt=fmt), nbytes=4 * n, name=f"k2_fmt{fmt}[{nm} {r}x{c}]")
        del e
    for nm, (r, c) in {"X": (8192, 4096), "H": (8192, 14336)}.items():
        a = torch.randn(r, c, generator=g, device=dev).to(bf)
        n = r * c
        for fmt in (0, 1, 2):
            timeit(lambda: halo.rotate_quantize(a, B, fmt=fmt), nbytes=3 * n, name=f"k1_fmt{fmt}[{nm} {r}x{c}]")
            timeit(lambda: halo.rotate_quantize(a, 1, fmt=fmt), nbytes=3 * n, name=f"k1_fmt{fmt}_B1[{nm} {r}x{c}]")
        del a
    # GEMM throughput per format (F shape of gate_proj, both operands K-major)
    M, N, K = 8192, 14336, 4096
    for fmt in (0, 1, 2):
        A = torch.randint(0, 64, (M, K), device=dev, dtype=torch.int32).to(torch.uint8) << 2
        Bm = torch.randint(0, 64, (N, K), device=dev, dtype=torch.int32).to(torch.uint8) << 2
        if fmt == 0:
            A, Bm = A.view(torch.int8), Bm.view(torch.int8)
        one = torch.ones(1, device=dev)
        timeit(lambda: halo.qmatmul(A, Bm, one, one, fmt=fmt, out="bf16"), ops=2.0 * M * N * K,
               name=f"gemm_fmt{fmt}[{M}x{N}x{K} bf16]")
        del A, Bm
