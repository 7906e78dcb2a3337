"""Generate golden fixtures from the REFERENCE itself (oracle/_ref, the
unmodified headers of /root/reference compiled by oracle/Makefile).

    python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Inputs come from the reference RNG
(tensor.hpp:398-445), rounded to bf16 the way the B200 path consumes them.
Run in the build container (needs /root/reference); the fixtures travel with
the repo so the GPU box can check against them without the reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402


def bf(a):
    return O.bf16_round(a)


def layer_inputs(b, m, n, seed):
    X = O.ref_randn(b, m, seed)
    X = O.ref_inject_outliers(X, [2, 9], 40.0)
    W = O.ref_randn(n, m, seed + 1, 1.0 / np.sqrt(m))
    E = O.ref_randn(b, n, seed + 2, 1e-3)
    E = O.ref_inject_outliers(E, [1, b // 2], 30.0, axis_rows=True)
    return bf(X), bf(W), bf(E)


def main():
    O.build()
    out = {}
    # ---- HaloLinearLayer end to end (halo_linear.hpp), full-dim (block 0)
    # and blocked transforms, INT8 and E4M3, every preset
    cases = [("halo0", 0, 0, 64, 64, 32), ("halo1", 0, 0, 64, 64, 32), ("halo2", 0, 0, 64, 64, 32),
             ("halo2", 0, 16, 48, 64, 32), ("halo2", 1, 0, 64, 64, 32), ("halo1", 1, 32, 64, 128, 64),
             ("halo2", 0, 64, 100, 128, 64)]
    for k, (name, fmt, block, b, m, n) in enumerate(cases):
        X, W, E = layer_inputs(b, m, n, 100 + k)
        lvl = {"halo0": 0, "halo1": 1, "halo2": 2}[name]
        r = O.ref_linear(lvl, fmt, block, X, W, E)
        np.savez_compressed(os.path.join(HERE, f"layer_{k}_{name}_fmt{fmt}_blk{block}.npz"), X=X, W=W, E=E,
                            level=lvl, fmt=fmt, block=block, **r)
        out[f"layer_{k}"] = (name, fmt, block, b, m, n)
    # ---- transforms and quantizers
    A = bf(O.ref_randn(24, 256, 7))
    np.savez_compressed(os.path.join(HERE, "transforms.npz"), A=A,
                        right_256=O.ref_fwht_rows(A, 256), right_16=O.ref_fwht_rows(A, 16),
                        left_8=O.ref_fwht_cols(A, 8))
    Q = O.ref_randn(33, 64, 9) * 3
    codes8, s8 = O.ref_quantize(Q, O.INT8)
    codes_e, se = O.ref_quantize(Q, O.FP8_E4M3)
    codes_r, sr = O.ref_quantize(Q, O.INT8, gran=1)
    codes_sup, _ = O.ref_quantize(Q, O.INT8, scales=np.array([0.05], np.float32))
    np.savez_compressed(os.path.join(HERE, "quantize.npz"), Q=Q, codes8=codes8, s8=s8, codes_e=codes_e, se=se,
                        codes_r=codes_r, sr=sr, codes_sup=codes_sup)
    # ---- HQ-FSDP protocol (hqfsdp.hpp)
    Wf = bf(O.ref_randn(10, 32, 11))
    fs = {}
    for world in (1, 2, 4, 8):
        codes, scale, am = O.ref_fsdp_gather(world, Wf, O.INT8, True)
        fs[f"codes_w{world}"] = codes
        fs[f"scale_w{world}"] = np.array([scale], np.float32)
        fs[f"absmax_w{world}"] = am
    G = O.ref_randn(4 * 10, 8, 12).reshape(4, 10, 8)
    fs["grads"] = G
    fs["rs"] = O.ref_reduce_scatter(G)
    np.savez_compressed(os.path.join(HERE, "fsdp.npz"), W=Wf, **fs)
    print("wrote", len(out), "layer fixtures + transforms/quantize/fsdp")


if __name__ == "__main__":
    main()
