"""cfg3 of BASELINE.json: HALO-1 vs HALO-2 FP8 (e4m3) full Llama-3-8B
transformer block fwd+bwd, seq 2048 x batch 8 (16384 tokens), one B200; plus
HALO-2 INT8 and the BF16 (cuBLAS) block for the speed-up the paper reports
(PAPER.md:755-756 measured these ratios on RTX 4090).  Synthetic data,
random-init weights.  CUDA-event timing, warm-up 3, L2 flushed between steps.

  python tools/bench_block.py [--steps 10] [--batch 8] [--seq 2048]
Prints one JSON line per configuration.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402
from paper_2501_02625_b200.block import LlamaBlock  # noqa: E402


def run(name, scheme, bf16, args):
    dev = torch.device("cuda", 0)
    blk = LlamaBlock(scheme, seq=args.seq, bf16=bf16)
    T = args.batch * args.seq
    g = torch.Generator(device=dev).manual_seed(1)
    x = torch.randn(T, 4096, generator=g, device=dev).to(torch.bfloat16)
    x[:, [2, 9, 16, 27]] *= 20
    dy = (torch.randn(T, 4096, generator=g, device=dev) * 1e-3).to(torch.bfloat16)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step():
        xi = x.detach().requires_grad_(True)
        y = blk.forward(xi)
        y.backward(dy)
        for l in blk.linears():
            l.grad = None
            l.w.grad = None  # bf16 arm: autograd's dW
        return xi.grad

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(args.steps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    ms = tot / args.steps
    ops = blk.gemm_ops(T)
    return {"config": name, "tokens": T, "ms_per_step": round(ms, 3), "tokens_per_s": round(T / ms * 1e3),
            "projection_gemm_TOPS_equiv": round(ops / ms / 1e9, 1),
            "note": "step = block forward + backward (5 projections, RMSNorm, RoPE, causal GQA SDPA attention)"}


def run_mlp(name, scheme, args):
    """Module-level comparison on cfg2's MLP (8192 tokens): HaloMLP (the
    bench.py path) vs the same MLP on bf16 cuBLAS linears with torch autograd."""
    import torch.nn.functional as F
    from paper_2501_02625_b200.mlp import HaloMLP
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    bf = torch.bfloat16
    H, I, T = 4096, 14336, 8192
    wg = (torch.randn(I, H, generator=g, device=dev) / H ** 0.5).to(bf)
    wu = (torch.randn(I, H, generator=g, device=dev) / H ** 0.5).to(bf)
    wd = (torch.randn(H, I, generator=g, device=dev) / I ** 0.5).to(bf)
    x = torch.randn(T, H, generator=g, device=dev).to(bf)
    dy = (torch.randn(T, H, generator=g, device=dev) * 1e-3).to(bf)
    if scheme is None:
        ws = [w.clone().requires_grad_(True) for w in (wg, wu, wd)]

        def step():
            xi = x.detach().requires_grad_(True)
            y = F.linear(F.silu(F.linear(xi, ws[0])) * F.linear(xi, ws[1]), ws[2])
            y.backward(dy)
            for w in ws:
                w.grad = None
    else:
        mlp = HaloMLP(wg, wu, wd, scheme)

        def step():
            mlp.forward(x)
            mlp.backward(dy)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(args.steps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    ms = tot / args.steps
    return {"config": "MLP " + name, "tokens": T, "ms_per_step": round(ms, 3), "tokens_per_s": round(T / ms * 1e3),
            "gemm_TOPS_equiv": round(6.0 * T * 3 * H * I / ms / 1e9, 1),
            "note": "cfg2 Llama-3-8B MLP fwd+bwd; bf16 = F.linear (cuBLAS) + torch autograd"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=2048)
    args = ap.parse_args()
    res = [run("bf16 (cuBLAS linears)", None, True, args),
           run("HALO-2 INT8 block 256", halo.halo2(halo.INT8, 256), False, args),
           run("HALO-1 FP8-E4M3 block 256", halo.halo1(halo.FP8_E4M3, 256), False, args),
           run("HALO-2 FP8-E4M3 block 256", halo.halo2(halo.FP8_E4M3, 256), False, args)]
    base = res[0]["ms_per_step"]
    for r in res:
        r["speedup_vs_bf16"] = round(base / r["ms_per_step"], 3)
        print(json.dumps(r), flush=True)
    mres = [run_mlp("bf16 (cuBLAS linears)", None, args), run_mlp("HALO-2 INT8 block 256", halo.halo2(halo.INT8, 256), args),
            run_mlp("HALO-2 FP8-E4M3 block 256", halo.halo2(halo.FP8_E4M3, 256), args)]
    for r in mres:
        r["speedup_vs_bf16"] = round(mres[0]["ms_per_step"] / r["ms_per_step"], 3)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
