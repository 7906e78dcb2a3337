"""HQ-FSDP over peer memory (csrc/peer.cu, halo_linear_set_qweight_sharded).

1. One process: (WH)_Q split into row shards held in separate buffers; the
   forward (B operand split along N) and E (operand split along the
   contracted dim) GEMMs read them through per-shard tensor maps.  Every
   output must equal the layer with the contiguous codes BIT-EXACTLY.
2. Two processes on the one GPU of the test box (gloo for the host-side
   handle exchange and the gradient reduce-scatter): shards exported by CUDA
   IPC, the absmax exchange and barriers through the device mailboxes
   (halo_peer_sync), GEMMs reading the peer's shard in place, G GEMMs
   storing their fp32 partial rows into the owner's receive buffer.  Each
   rank's outputs equal the single-process HaloMLP on its tokens bit for bit,
   and each gradient shard equals the rank-order double mean of the per-rank
   fp32 gradients (reduce_scatter_grads, hqfsdp.hpp:271-300) bit for bit.
"""
import os
import socket

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_02625_b200 import halo
    return halo


def _w(n, m, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = (torch.randn(n, m, generator=g, device="cuda") / m ** 0.5)
    w[:, 3] *= 20
    return w.to(torch.bfloat16), g


@pytest.mark.parametrize("scheme", ["halo2", "halo1", "halo0"])
@pytest.mark.parametrize("fmt", [0, 1])
@pytest.mark.parametrize("parts", [2, 4])
def test_sharded_qweight_bitexact(H, scheme, fmt, parts):
    n, m, b = 1024, 512, 384
    w, g = _w(n, m, 11)
    x = torch.randn(b, m, generator=g, device="cuda").to(torch.bfloat16)
    e = (torch.randn(b, n, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    sch = H.scheme_from_string(scheme, fmt, 256)
    ref = H.HaloLinearLayer(w, sch, out_dtype=torch.float32, grad_dtype=torch.float32)
    rc = H.SavedContext()
    y0 = ref.forward(x, rc)
    b0 = ref.backward(rc, e)
    # the (W[H])_Q the layer quantized itself: the exported inference
    # weights (halo_linear.hpp:332-338) for the rotated schemes, the plain
    # per-tensor codes for HALO-0
    if sch.F.middle:
        codes, scale = ref.export_inference_weights()
    else:
        codes, scale = H.rotate_quantize(w, 1, fmt, rotate=False)
    rows = n // parts
    shards = [codes[i * rows:(i + 1) * rows].clone() for i in range(parts)]  # separate allocations
    lay = H.HaloLinearLayer(w, sch, out_dtype=torch.float32, grad_dtype=torch.float32)
    lay.set_qweight_sharded(shards, scale)
    c = H.SavedContext()
    y1 = lay.forward(x, c)
    b1 = lay.backward(c, e)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    assert torch.equal(b0.e_x, b1.e_x)
    assert torch.equal(b0.grad_w, b1.grad_w)


def test_sharded_qweight_rejects_bad_split(H):
    w, _ = _w(768, 256, 3)
    lay = H.HaloLinearLayer(w, H.halo2(0, 256))
    codes = torch.zeros(768, 256, dtype=torch.int8, device="cuda")
    scale = torch.ones(1, device="cuda")
    with pytest.raises(ValueError):
        lay.set_qweight_sharded([codes[:384], codes[384:]], scale)  # 384 rows: not a multiple of 256


@pytest.mark.parametrize("scheme", ["halo2", "halo1", "halo0"])
@pytest.mark.parametrize("parts,rank", [(1, 0), (2, 1), (4, 2)])
def test_grad_scatter_single_process(H, scheme, parts, rank):
    """The G GEMM's fp32 rows land in slot `rank` of each owner's receive
    buffer (all local here), equal to the layer's own fp32 grad_w."""
    from paper_2501_02625_b200._lib import check, lib
    n, m, b = 1024, 512, 384
    w, g = _w(n, m, 21)
    x = torch.randn(b, m, generator=g, device="cuda").to(torch.bfloat16)
    e = (torch.randn(b, n, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    sch = H.scheme_from_string(scheme, 0, 256)
    ref = H.HaloLinearLayer(w, sch, out_dtype=torch.float32, grad_dtype=torch.float32)
    rc = H.SavedContext()
    ref.forward(x, rc)
    b0 = ref.backward(rc, e)
    rows = n // parts
    recv = [torch.full((parts, rows, m), float("nan"), device="cuda") for _ in range(parts)]
    lay = H.HaloLinearLayer(w, sch, out_dtype=torch.float32, grad_dtype=torch.float32)
    lay.set_grad_scatter([r.data_ptr() for r in recv], rank)
    c = H.SavedContext()
    lay.forward(x, c)
    b1 = lay.backward(c, e)
    assert b1.grad_w is None
    torch.cuda.synchronize()
    assert torch.equal(b0.e_x, b1.e_x)
    for i in range(parts):
        assert torch.equal(recv[i][rank], b0.grad_w[i * rows:(i + 1) * rows])
    # owner side: rank-order double mean (hqfsdp.hpp:288-292)
    box = torch.stack([b0.grad_w[:rows], (b0.grad_w[:rows] * 3).contiguous()])
    out = torch.empty(rows, m, device="cuda")
    check(lib().halo_reduce_scatter_shard(H._ptr(box), 2, rows, m, H._ptr(out), 0, H._stream()))
    torch.cuda.synchronize()
    want = ((box[0].double() + box[1].double()) / 2).float()
    assert torch.equal(out, want)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mlp_data(rank=0, H=512, I=1024, T=512):
    """Shards of 256 (down) and 512 (gate/up) rows at world 2; weights
    shared, tokens per rank."""
    g = torch.Generator(device="cuda").manual_seed(0)
    bf = torch.bfloat16
    wg = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
    wu = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
    wd = (torch.randn(H, I, generator=g, device="cuda") / I ** 0.5).to(bf)
    g = torch.Generator(device="cuda").manual_seed(100 + rank)
    x = torch.randn(T, H, generator=g, device="cuda").to(bf)
    x[:, [2, 9]] *= 30
    dy = (torch.randn(T, H, generator=g, device="cuda") * 1e-3).to(bf)
    return wg, wu, wd, x, dy


def _peer_worker(rank, world, port, out_dir, staged=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_02625_b200 import halo
    from paper_2501_02625_b200.fsdp import PeerFsdpHaloMLP
    wg, wu, wd, x, dy = _mlp_data(rank)
    mlp = PeerFsdpHaloMLP(wg, wu, wd, halo.halo2(0, 256), grad_dtype=torch.float32, staged=staged)
    outs = []
    for _ in range(2):  # two steps: the second re-quantizes shards peers read in the first
        y = mlp.forward(x)
        dx, shards = mlp.backward(dy)
        torch.cuda.synchronize()
        outs.append((y.cpu(), dx.cpu(), [s.cpu() for s in shards]))
    torch.save({"rank": rank, "outs": outs, "ledger_gather": mlp.ledger.gather.payload}, os.path.join(out_dir, f"r{rank}.pt"))
    dist.barrier()
    mlp.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("staged", [False, True])
def test_peer_fsdp_two_processes(H, tmp_path, staged):
    """In-place peer reads and the staged copy (one NVLink copy of each peer
    shard per step) give the same bits as the single-process MLP."""
    import torch.multiprocessing as mp
    from paper_2501_02625_b200.mlp import HaloMLP
    world = 2
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, str(tmp_path), staged)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    for p in procs:
        if p.is_alive():
            p.kill()
            p.join()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    # single-process reference per rank's tokens; the shards are the
    # rank-order double mean of the per-rank fp32 gradients
    per = []
    for r in range(world):
        wg, wu, wd, x, dy = _mlp_data(r)
        ref = HaloMLP(wg, wu, wd, H.halo2(0, 256))
        for l in (ref.gate, ref.up, ref.down):
            l.grad_dtype = torch.float32
        y = ref.forward(x)
        dx, grads = ref.backward(dy)
        torch.cuda.synchronize()
        per.append((y.cpu(), dx.cpu(), [gr.cpu() for gr in grads]))
    mean = [((per[0][2][i].double() + per[1][2][i].double()) / 2).float() for i in range(3)]
    for r in range(world):
        res = torch.load(os.path.join(str(tmp_path), f"r{r}.pt"))
        for (py, pdx, pshards) in res["outs"]:
            assert torch.equal(py, per[r][0])
            assert torch.equal(pdx, per[r][1])
            for gm, gs in zip(mean, pshards):
                rows = gs.shape[0]
                assert torch.equal(gs, gm[r * rows:(r + 1) * rows])
