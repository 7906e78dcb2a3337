"""HQ-FSDP protocol on real ranks: world_size 2 and 4 over gloo on CPU.

The protocol code (paper_2501_02625_b200/fsdp.py) runs unchanged; the device
ops are replaced by the CPU oracle (the checker) so the collectives, the
padding, the shared-scale agreement, the regather and the stale check are
exercised here.  Mirrors test_hqfsdp.cpp:84-257.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleOps:
    """CPU stand-in for the K1 kernels (test infrastructure only)."""

    def __init__(self, O):
        self.O = O

    def absmax(self, a, had_block, rotate):
        x = a.float().numpy()
        if rotate:
            x = self.O.fwht_rows(x, had_block or x.shape[1])
        return torch.tensor([float(np.abs(x).max()) if x.size else 0.0], dtype=torch.float32)

    def quantize(self, a, had_block, fmt, scale, rotate):
        x = a.float().numpy()
        if rotate:
            x = self.O.fwht_rows(x, had_block or x.shape[1])
        codes, _ = self.O.quantize(x, fmt, scales=scale.numpy().astype(np.float32))
        return torch.from_numpy(self.O.codes_to_bytes(codes, fmt).view(np.int8).copy())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2501_02625_b200 import fsdp
        from paper_2501_02625_b200._lib import HaloLogicError
        ops = OracleOps(O)
        out = {}
        # 10 x 32 weight: rows pad to 10 (w=2) or 12 (w=4) (test_hqfsdp.cpp:47-70)
        W = torch.from_numpy(O.bf16_round(O.randn(10, 32, 7)))
        for fmt in (fsdp.INT8, fsdp.FP8_E4M3):
            p = fsdp.shard(W, fsdp.WorldConfig(world), fmt, rank)
            ledger = fsdp.CommLedger()
            codes, scale = fsdp.quantized_all_gather(p, True, ledger, 0, ops=ops)
            out[f"codes{fmt}"] = codes.numpy().copy()
            out[f"scale{fmt}"] = float(scale)
            out[f"absmax{fmt}"] = [float(v) for v in p.local_absmax]
            sr = ledger.scale_reduce.payload
            again, _ = fsdp.backward_regather(p, True, ledger, True, 0, ops=ops)
            out[f"regather_equal{fmt}"] = bool(torch.equal(again, codes))
            out[f"no_scale_traffic{fmt}"] = ledger.scale_reduce.payload == sr
            out[f"ratio{fmt}"] = fsdp.comm_report(ledger).gather_ratio_vs_bf16
            # stale weights are detected on every rank (test_hqfsdp.cpp:175-179)
            if rank == 0:
                p.master[0, 0] += 10.0
            try:
                fsdp.backward_regather(p, True, ledger, True, 0, ops=ops)
                out[f"stale{fmt}"] = False
            except HaloLogicError:
                out[f"stale{fmt}"] = True
        # regather without a forward gather is a logic error
        p = fsdp.shard(W, fsdp.WorldConfig(world), fsdp.INT8, rank)
        try:
            fsdp.backward_regather(p, True, fsdp.CommLedger(), ops=ops)
            out["missing"] = False
        except HaloLogicError:
            out["missing"] = True
        # reduce-scatter of per-rank gradients (test_hqfsdp.cpp:182-224)
        G = torch.from_numpy(O.randn(10, 8, 100 + rank))
        shard_grad = fsdp.reduce_scatter_grads(G, fsdp.shard(torch.zeros(10, 8), fsdp.WorldConfig(world),
                                                             fsdp.INT8, rank), fsdp.CommLedger())
        out["rs"] = shard_grad.numpy().copy()
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_hqfsdp_protocol_gloo(orc, world):
    O = orc
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), results), nprocs=world, join=True, start_method="spawn")
    W = O.bf16_round(O.randn(10, 32, 7))
    padded = (10 + world - 1) // world * world
    P = np.zeros((padded, 32), np.float32)
    P[:10] = W
    rot = O.fwht_rows(P, 32)
    for fmt in (0, 1):
        want_codes, want_s = O.quantize(rot, fmt)
        want = O.codes_to_bytes(want_codes, fmt).view(np.int8)
        for r in range(world):
            res = results[r]
            # gather == single-process quantization of the padded rotated weight
            assert np.array_equal(res[f"codes{fmt}"], want)
            assert res[f"scale{fmt}"] == want_s[0]
            assert res[f"regather_equal{fmt}"] and res[f"no_scale_traffic{fmt}"]
            assert res[f"stale{fmt}"]
            assert abs(res[f"ratio{fmt}"] - 0.5) < 5e-4 + 4.0 / (2 * padded * 32)
        # per-rank absmax of the rotated shards, max-reduced
        shard_rows = padded // world
        ams = [float(np.abs(rot[r * shard_rows:(r + 1) * shard_rows]).max()) for r in range(world)]
        assert results[0][f"absmax{fmt}"] == pytest.approx(ams, rel=0, abs=0)
    assert all(results[r]["missing"] for r in range(world))
    # mean of the per-rank gradients, scattered by rows; world 2 is exact
    G = np.stack([O.randn(10, 8, 100 + r) for r in range(world)])
    mean = (G.astype(np.float64).sum(0) / world).astype(np.float32)
    shard_rows = (10 + world - 1) // world
    got = np.concatenate([results[r]["rs"] for r in range(world)])[:10]
    if world == 2:
        assert np.array_equal(got, mean)
    else:
        assert np.allclose(got, mean, rtol=1e-6, atol=1e-7)


def test_fp6_payload_ratio():
    """hqfsdp.hpp:36-49 / test_hqfsdp.cpp:245-257: FP6 packs 4 codes into 3
    bytes -- 0.375 of BF16 (INT8 / FP8: 0.5)."""
    from paper_2501_02625_b200 import fsdp
    n = 256 * 64
    assert fsdp.code_payload_bytes(fsdp.FP6_E3M2, n) == 12288
    assert fsdp.code_payload_bytes(fsdp.FP6_E3M2, n) / (2 * n) == 0.375
    assert fsdp.code_payload_bytes(fsdp.INT8, n) / (2 * n) == 0.5
    assert fsdp.code_payload_bytes(fsdp.FP6_E3M2, 5) == 6  # (5 + 3) // 4 * 3

