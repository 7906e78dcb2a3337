"""HQ-FSDP (hqfsdp.hpp) on real ranks: one process per GPU, NCCL over NVLink.

The reference simulates the protocol with logical ranks in one process
(hqfsdp.hpp:3-10).  Here every rank owns a contiguous row shard of each
linear weight (rows zero-padded to a multiple of the world size,
hqfsdp.hpp:131-148) and the collectives are real:

  forward gather   (hqfsdp.hpp:204-237)  local rotate + absmax (K1 phase A on
                   the shard) -> all-gather of the per-rank absmax (max is
                   order-insensitive) -> shared scale float(max/fmax) ->
                   local quantize under that scale (K1 phase B) ->
                   all-gather of the INT8/E4M3 codes
  backward regather (:243-266)           same codes under the SAVED scale, no
                   scale traffic; optional stale-weight check
  reduce-scatter   (:271-300)            dW summed over ranks and scattered
                   by row range, divided by the world size

Because per-tensor scales are shared, the gathered codes equal a
single-process quantization of the rotated padded weight bit for bit
(test_hqfsdp.cpp:98-125); the gradient mean is fp32 in NCCL order instead of
the reference's double rank-order sum (tolerance parity).

The byte ledger (:36-103) is kept so the reference's compression ratios
(INT8 gather = 0.5 x BF16) can be reported.  Device work goes through an
``ops`` object: the default is the CUDA path of this package; the CPU
multi-process tests inject a checker implementation.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from ._lib import HaloLogicError

INT8, FP8_E4M3, FP6_E3M2 = 0, 1, 2
_FMAX = {INT8: 127.0, FP8_E4M3: 448.0, FP6_E3M2: 28.0}
K_SCALE_BYTES = 4  # hqfsdp.hpp:55


# ------------------------------------------------------------ byte model --

def code_payload_bytes(fmt: int, elems: int) -> int:
    """hqfsdp.hpp:36-49: INT8/FP8 one byte per code, FP6 four codes in three
    bytes (the wire format; the device keeps one code per byte)."""
    if fmt in (INT8, FP8_E4M3):
        return elems
    if fmt == FP6_E3M2:
        return (elems + 3) // 4 * 3
    raise ValueError("only int8 / fp8_e4m3 / fp6_e3m2 payloads are on the device path")


@dataclass
class CollectiveStat:  # hqfsdp.hpp:57-61
    payload: int = 0
    transferred: int = 0
    count: int = 0


@dataclass
class CommLedger:  # hqfsdp.hpp:65-79
    gather: CollectiveStat = field(default_factory=CollectiveStat)
    scale_reduce: CollectiveStat = field(default_factory=CollectiveStat)
    reduce_scatter: CollectiveStat = field(default_factory=CollectiveStat)
    bf16_gather_payload: int = 0
    backward_gathers: int = 0
    backward_consumers: int = 0

    def record(self, c: CollectiveStat, payload: int, world: int):
        c.payload += payload
        c.transferred += payload * (world - 1) // world
        c.count += 1


@dataclass
class CommReport:  # hqfsdp.hpp:81-103
    gather_payload: int
    gather_transferred: int
    scale_reduce_payload: int
    scale_reduce_transferred: int
    reduce_scatter_payload: int
    reduce_scatter_transferred: int
    gather_ratio_vs_bf16: float


def comm_report(ledger: CommLedger) -> CommReport:
    ratio = ledger.gather.payload / ledger.bf16_gather_payload if ledger.bf16_gather_payload else 1.0
    return CommReport(ledger.gather.payload, ledger.gather.transferred, ledger.scale_reduce.payload,
                      ledger.scale_reduce.transferred, ledger.reduce_scatter.payload,
                      ledger.reduce_scatter.transferred, ratio)


# --------------------------------------------------------------- devices --

class CudaOps:
    """The B200 kernels (K1 phase A / phase B) behind the protocol."""

    def absmax(self, a: torch.Tensor, had_block: int, rotate: bool) -> torch.Tensor:
        from . import halo
        return halo.rotate_absmax(a, had_block, rotate)

    def quantize(self, a: torch.Tensor, had_block: int, fmt: int, scale: torch.Tensor, rotate: bool, out=None):
        from . import halo
        codes, _ = halo.rotate_quantize(a, had_block, fmt, scale=scale, rotate=rotate, out=out)
        return codes


class NcclDataPlane:
    """The C++ HQ-FSDP data plane of this rank (halo_fsdp_*, csrc/hqfsdp_nccl.cpp:
    NCCL resolved at run time): quantized_all_gather / backward_regather /
    reduce_scatter_grads as stream-ordered library calls, no host syncs.  The
    communicator's unique id is broadcast over `group` (any backend); with
    torch.distributed uninitialised it is a world of one."""

    def __init__(self, group=None):
        import ctypes as C
        from ._lib import check, lib
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = (C.c_char * 128)()
        if self.rank == 0:
            check(lib().halo_fsdp_get_unique_id(uid))
        if self.world > 1:
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            uid = (C.c_char * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        check(lib().halo_fsdp_create(uid, self.world, self.rank, C.byref(h)))
        self._h = h

    def close(self):
        from ._lib import lib
        if getattr(self, "_h", None):
            lib().halo_fsdp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    @staticmethod
    def _blk(p, rotate, had_block):
        return had_block if rotate else -1

    def gather(self, p: "ShardedParam", rotate: bool, had_block: int, out: torch.Tensor, ledger: "CommLedger"):
        """quantized_all_gather (hqfsdp.hpp:204-237) into `out`."""
        from . import halo
        from ._lib import check, lib
        if p.local_absmax is None or p.local_absmax.numel() != 1:
            p.local_absmax = torch.empty(1, dtype=torch.float32, device=p.master.device)
        if p.global_scale is None or p.global_scale.numel() != 1:
            p.global_scale = torch.empty(1, dtype=torch.float32, device=p.master.device)
        check(lib().halo_fsdp_quantized_all_gather(self._h, halo._ptr(p.master), halo._dt(p.master), p.shard_rows,
                                                   p.cols, self._blk(p, rotate, had_block), p.format, halo._ptr(out),
                                                   halo._ptr(p.global_scale), halo._ptr(p.local_absmax),
                                                   halo._stream()))
        p.scales_valid = True
        ledger.record(ledger.scale_reduce, K_SCALE_BYTES, p.world)
        elems = out.numel()
        ledger.record(ledger.gather, code_payload_bytes(p.format, elems) + K_SCALE_BYTES, p.world)
        ledger.bf16_gather_payload += 2 * elems
        return out, p.global_scale

    def regather(self, p: "ShardedParam", rotate: bool, had_block: int, out: torch.Tensor, ledger: "CommLedger",
                 stale_flag: torch.Tensor | None = None):
        """backward_regather (hqfsdp.hpp:243-266); stale_flag: int32 [1]."""
        from . import halo
        from ._lib import check, lib
        if not p.scales_valid:
            raise HaloLogicError("backward_regather: no saved forward scales")
        check(lib().halo_fsdp_backward_regather(self._h, halo._ptr(p.master), halo._dt(p.master), p.shard_rows,
                                                p.cols, self._blk(p, rotate, had_block), p.format,
                                                halo._ptr(p.global_scale),
                                                halo._ptr(p.local_absmax) if stale_flag is not None else None,
                                                halo._ptr(stale_flag), halo._ptr(out), halo._stream()))
        ledger.backward_gathers += 1
        elems = out.numel()
        ledger.record(ledger.gather, code_payload_bytes(p.format, elems) + K_SCALE_BYTES, p.world)
        ledger.bf16_gather_payload += 2 * elems
        return out, p.global_scale

    def reduce_scatter(self, grad: torch.Tensor, p: "ShardedParam", ledger: "CommLedger") -> torch.Tensor:
        """reduce_scatter_grads (hqfsdp.hpp:271-300): this rank's rows of the mean."""
        from . import halo
        from ._lib import check, lib
        if tuple(grad.shape) != (p.full_rows, p.cols):
            raise ValueError("reduce_scatter_grads: gradient shape mismatch")
        if p.world == 1 and p.pad_rows == 0:
            ledger.record(ledger.reduce_scatter, 2 * grad.numel(), 1)
            return grad
        if p.pad_rows:
            padded = torch.zeros((p.shard_rows * p.world, p.cols), dtype=grad.dtype, device=grad.device)
            padded[: p.full_rows] = grad
        else:
            padded = grad.contiguous()
        out = torch.empty((p.shard_rows, p.cols), dtype=grad.dtype, device=grad.device)
        check(lib().halo_fsdp_reduce_scatter(self._h, halo._ptr(padded), halo._dt(padded), p.shard_rows, p.cols,
                                             halo._ptr(out), halo._stream()))
        ledger.record(ledger.reduce_scatter, 2 * padded.numel(), p.world)
        return out

    def all_reduce_mean(self, t: torch.Tensor):
        from . import halo
        from ._lib import check, lib
        check(lib().halo_fsdp_all_reduce_mean(self._h, halo._ptr(t), halo._dt(t), t.numel(), halo._stream()))
        return t


# ------------------------------------------------------------- sharding --

@dataclass
class WorldConfig:  # hqfsdp.hpp:26-30
    world_size: int = 1
    shard_linear: bool = True
    replicate_norms: bool = True


@dataclass
class ShardedParam:  # hqfsdp.hpp:107-120
    master: torch.Tensor          # this rank's rows of the padded weight
    full_rows: int
    pad_rows: int
    world: int
    rank: int
    shard_rows: int
    cols: int
    format: int = INT8
    local_absmax: torch.Tensor | None = None  # one per rank, over the rotated shard
    global_scale: torch.Tensor | None = None
    scales_valid: bool = False


def row_range(p: ShardedParam, rank: int):
    """hqfsdp.hpp:122-125"""
    return rank * p.shard_rows, (rank + 1) * p.shard_rows


def shard(w: torch.Tensor, world: WorldConfig, fmt: int, rank: int) -> ShardedParam:
    """hqfsdp.hpp:131-148: rows padded with zeros to a multiple of the world
    size; rank r keeps rows [r*shard_rows, (r+1)*shard_rows)."""
    if world.world_size < 1:
        raise ValueError("shard: world_size must be at least 1")
    rows, cols = w.shape
    padded = (rows + world.world_size - 1) // world.world_size * world.world_size
    shard_rows = padded // world.world_size
    local = torch.zeros((shard_rows, cols), dtype=w.dtype, device=w.device)
    lo = rank * shard_rows
    hi = min(rows, lo + shard_rows)
    if hi > lo:
        local[: hi - lo] = w[lo:hi]
    return ShardedParam(local, rows, padded - rows, world.world_size, rank, shard_rows, cols, fmt)


def scale_from_absmax(m: torch.Tensor, fmt: int) -> torch.Tensor:
    """hqfsdp.hpp:172-177 / quantize.hpp:234: float(double(m)/fmax), 1 if 0."""
    s = (m.double() / _FMAX[fmt]).float()
    return torch.where(m == 0, torch.ones_like(s), s)


def _gather(t: torch.Tensor, group, out: torch.Tensor | None = None) -> torch.Tensor:
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    shape = (world * t.shape[0],) + tuple(t.shape[1:])
    if out is None:
        out = torch.empty(shape, dtype=t.dtype, device=t.device)
    elif tuple(out.shape) != shape or out.dtype != t.dtype:
        raise ValueError("gather: output buffer shape/dtype mismatch")
    if world == 1:
        out.copy_(t)
    elif dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    else:
        dist.all_gather(list(out.chunk(world, 0)), t.contiguous(), group=group)
    return out


def quantized_all_gather(p: ShardedParam, apply_hadamard: bool, ledger: CommLedger, had_block: int = 0,
                         group=None, ops=None, out: torch.Tensor | None = None):
    """Forward gather (hqfsdp.hpp:204-237).  Returns (codes, scale): the
    (rows_padded x cols) codes and the shared per-tensor scale, identical on
    every rank."""
    ops = ops or CudaOps()
    am = ops.absmax(p.master, had_block, apply_hadamard).reshape(1).float()
    all_am = _gather(am, group)  # every rank's local absmax, kept (on device) for the stale check
    p.local_absmax = all_am
    g = all_am.max().reshape(1)
    p.global_scale = scale_from_absmax(g, p.format)
    p.scales_valid = True
    ledger.record(ledger.scale_reduce, K_SCALE_BYTES, p.world)
    return _gather_with_scale(p, apply_hadamard, ledger, had_block, group, ops, out)


def _gather_with_scale(p, apply_hadamard, ledger, had_block, group, ops, out=None):
    """hqfsdp.hpp:184-196: quantize the local rotated rows under the agreed
    scale, gather the codes, book the bytes."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1 and out is not None and isinstance(ops, CudaOps):
        # a world of one: the local codes ARE the gathered tensor
        full = ops.quantize(p.master, had_block, p.format, p.global_scale, apply_hadamard, out=out.view(p.master.shape))
    else:
        codes = ops.quantize(p.master, had_block, p.format, p.global_scale, apply_hadamard)
        full = _gather(codes, group, out)
    elems = full.numel()
    ledger.record(ledger.gather, code_payload_bytes(p.format, elems) + K_SCALE_BYTES, p.world)
    ledger.bf16_gather_payload += 2 * elems
    return full, p.global_scale


def backward_regather(p: ShardedParam, apply_hadamard: bool, ledger: CommLedger, check_stale: bool = True,
                      had_block: int = 0, group=None, ops=None, out: torch.Tensor | None = None,
                      stale_flag: torch.Tensor | None = None):
    """Backward gather under the saved forward scale (hqfsdp.hpp:243-266).
    stale_flag (device fp32 [1]): the stale-weight check is accumulated
    there without a host sync (the caller reduces and tests it once, see
    check_stale_flag); otherwise it raises here."""
    if not p.scales_valid:
        raise HaloLogicError("backward_regather: no saved forward scales")
    ops = ops or CudaOps()
    if check_stale and stale_flag is not None:
        am = ops.absmax(p.master, had_block, apply_hadamard).reshape(1).float()
        saved = p.local_absmax[p.rank].reshape(1).float() if p.local_absmax.numel() > 1 else p.local_absmax.reshape(1)
        torch.maximum(stale_flag, (am != saved).float(), out=stale_flag)
    elif check_stale:
        am = float(ops.absmax(p.master, had_block, apply_hadamard).reshape(-1)[0])
        stale = torch.tensor([1.0 if am != float(p.local_absmax[p.rank]) else 0.0])
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            stale = stale.to(p.master.device)
            dist.all_reduce(stale, op=dist.ReduceOp.MAX, group=group)
        if float(stale) != 0.0:
            raise HaloLogicError("backward_regather: saved scales are stale (weights changed since the forward gather)")
    ledger.backward_gathers += 1
    return _gather_with_scale(p, apply_hadamard, ledger, had_block, group, ops, out)


def check_stale_flag(stale_flag: torch.Tensor, group=None):
    """Raise HaloLogicError if any rank's accumulated stale flag is set
    (backward_regather's check, hqfsdp.hpp:256-259, reduced once)."""
    f = stale_flag.clone()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(f, op=dist.ReduceOp.MAX, group=group)
    if float(f.item()) != 0.0:
        raise HaloLogicError("backward_regather: saved scales are stale (weights changed since the forward gather)")


def reduce_scatter_grads(grad: torch.Tensor, p: ShardedParam, ledger: CommLedger, group=None) -> torch.Tensor:
    """hqfsdp.hpp:271-300: mean over ranks, scattered by row range.  `grad`
    is this rank's full (rows x cols) gradient; padding rows are zero and the
    returned shard has shard_rows rows (rows past full_rows stay zero)."""
    if tuple(grad.shape) != (p.full_rows, p.cols):
        raise ValueError("reduce_scatter_grads: gradient shape mismatch")
    world = p.world
    if p.pad_rows == 0:
        if world == 1:  # a world of one owns every row: the mean is the gradient itself
            ledger.record(ledger.reduce_scatter, 2 * grad.numel(), world)
            return grad
        padded = grad.contiguous()
    else:
        padded = torch.zeros((p.shard_rows * p.world, p.cols), dtype=grad.dtype, device=grad.device)
        padded[: p.full_rows] = grad
    out = torch.empty((p.shard_rows, p.cols), dtype=grad.dtype, device=grad.device)
    if world == 1:
        out.copy_(padded)
    elif dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, padded, op=dist.ReduceOp.SUM, group=group)
        out.div_(world)
    else:  # gloo has no reduce_scatter: all-reduce then slice
        if padded is grad:
            padded = grad.clone()  # never sum into the caller's gradient
        dist.all_reduce(padded, op=dist.ReduceOp.SUM, group=group)
        out.copy_(padded[p.rank * p.shard_rows:(p.rank + 1) * p.shard_rows])
        out.div_(world)
    ledger.record(ledger.reduce_scatter, 2 * padded.numel(), world)
    return out


class FsdpHaloMLP:
    """Llama MLP block (mlp.HaloMLP) with HQ-FSDP weights: each rank keeps a
    row shard of gate/up/down; every step gathers the INT8 (WH)_Q codes for
    the forward, regathers them for the backward under the saved scale, and
    reduce-scatters the weight gradients (the loop of hqfsdp.hpp:361-411).

    data_plane="native" runs the collectives through the library's C++ NCCL
    data plane (NcclDataPlane, halo_fsdp_*), "torch" through the protocol
    functions above on torch.distributed.  With `overlap` the gathers /
    regathers of all three weights are issued up front on a side stream and
    each projection waits only for its own codes; each dW reduce-scatter
    starts on that stream as soon as its G GEMM is done, behind the next
    projection's backward."""

    def __init__(self, w_gate, w_up, w_down, scheme, group=None, check_stale=False, grad_dtype=torch.bfloat16,
                 data_plane: str | None = "native", overlap: bool = True):
        from .mlp import HaloMLP
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.fmt = scheme.format_w
        self.block = scheme.had_block
        self.rotate = bool(scheme.F.middle)
        self.check_stale = check_stale
        self.params = [shard(w, WorldConfig(self.world), self.fmt, self.rank) for w in (w_gate, w_up, w_down)]
        self.mlp = HaloMLP(w_gate, w_up, w_down, scheme)
        for layer in self.layers:
            layer.grad_dtype = grad_dtype
        code_dt = torch.int8 if self.fmt == INT8 else torch.uint8
        self.buffers = [torch.empty((p.shard_rows * p.world, p.cols), dtype=code_dt, device=p.master.device)
                        for p in self.params]
        self.ledger = CommLedger()
        self.plane = NcclDataPlane(group) if data_plane == "native" else None
        dev = self.params[0].master.device
        self.overlap = overlap
        self.comm = torch.cuda.Stream(device=dev) if overlap else None
        self.ready = {n: torch.cuda.Event() for n in ("gate", "up", "down")}
        self.stale = torch.zeros(1, dtype=torch.int32 if self.plane else torch.float32, device=dev)
        self._shards = {}

    @property
    def layers(self):
        return (self.mlp.gate, self.mlp.up, self.mlp.down)

    _IDX = {"gate": 0, "up": 1, "down": 2}

    def _install(self, layer, codes, scale, rows):
        layer.set_qweight(codes[:rows], scale)

    def _fetch_all(self, regather: bool, order):
        main = torch.cuda.current_stream()
        side = self.comm if self.overlap else main
        side.wait_stream(main)  # masters written / buffers last read before this point
        with torch.cuda.stream(side):
            for name in order:
                i = self._IDX[name]
                p, buf, layer = self.params[i], self.buffers[i], self.layers[i]
                if regather:
                    if self.plane is not None:
                        codes, scale = self.plane.regather(p, self.rotate, self.block, buf, self.ledger,
                                                           self.stale if self.check_stale else None)
                    else:
                        codes, scale = backward_regather(p, self.rotate, self.ledger, self.check_stale, self.block,
                                                         self.group, out=buf)
                    self.ledger.backward_consumers += 1
                elif self.plane is not None:
                    codes, scale = self.plane.gather(p, self.rotate, self.block, buf, self.ledger)
                else:
                    codes, scale = quantized_all_gather(p, self.rotate, self.ledger, self.block, self.group, out=buf)
                self._install(layer, codes, scale, p.full_rows)
                self.ready[name].record(side)

    def _wait(self, name, phase):
        torch.cuda.current_stream().wait_event(self.ready[name])

    def _rs(self, name, grad):
        i = self._IDX[name]
        p = self.params[i]
        if grad is None:
            return None
        main = torch.cuda.current_stream()
        side = self.comm if self.overlap else main
        side.wait_stream(main)  # the G GEMM wrote grad
        with torch.cuda.stream(side):
            if self.plane is not None:
                out = self.plane.reduce_scatter(grad, p, self.ledger)
            else:
                out = reduce_scatter_grads(grad, p, self.ledger, self.group)
            grad.record_stream(side)
            out.record_stream(side)
        return out

    def forward(self, x):
        if self.plane is not None and self.check_stale:
            self.stale.zero_()
        self._fetch_all(False, ("gate", "up", "down"))
        self.mlp.pre = self._wait
        self.mlp.post_grad = None
        return self.mlp.forward(x)

    def backward(self, dy):
        self._fetch_all(True, ("down", "gate", "up"))
        self.mlp.pre = self._wait
        self.mlp.post_grad = self._rs
        dx, shards = self.mlp.backward(dy)
        if self.overlap:
            torch.cuda.current_stream().wait_stream(self.comm)
        if self.plane is not None and self.check_stale:
            check_stale_flag(self.stale, self.group)
        return dx, list(shards)

    def gemm_ops(self, tokens):
        return self.mlp.gemm_ops(tokens)

    def close(self):
        torch.cuda.synchronize()
        if self.plane is not None:
            self.plane.close()


# ------------------------------------------------- peer-memory HQ-FSDP --

class PeerBuffer:
    """A device buffer from halo_peer_alloc (zero-filled, exportable by CUDA
    IPC), optionally viewed as a torch tensor through the CUDA array
    interface."""

    _TYPESTR = {torch.int8: "|i1", torch.uint8: "|u1", torch.float32: "<f4"}

    def __init__(self, nbytes: int):
        import ctypes as C
        from ._lib import check, lib
        p = C.c_void_p()
        check(lib().halo_peer_alloc(nbytes, C.byref(p)))
        self.ptr, self.nbytes = p.value, nbytes

    def tensor(self, shape, dtype) -> torch.Tensor:
        ptr = self.ptr

        class _View:
            __cuda_array_interface__ = {"shape": tuple(shape), "typestr": PeerBuffer._TYPESTR[dtype],
                                        "data": (ptr, False), "version": 2, "strides": None}

        return torch.as_tensor(_View(), device=torch.device("cuda", torch.cuda.current_device()))

    def handle(self) -> bytes:
        import ctypes as C
        from ._lib import check, lib
        buf = C.create_string_buffer(64)
        check(lib().halo_ipc_handle(C.c_void_p(self.ptr), buf))
        return buf.raw

    def free(self):
        from ._lib import lib
        if self.ptr:
            lib().halo_peer_free(self.ptr)
            self.ptr = 0


def _ipc_open(handle: bytes) -> int:
    import ctypes as C
    from ._lib import check, lib
    p = C.c_void_p()
    check(lib().halo_ipc_open(handle, C.byref(p)))
    return p.value


def _exchange(obj, group):
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return [obj]
    out = [None] * world
    dist.all_gather_object(out, obj, group=group)
    return out


class PeerFsdpHaloMLP(FsdpHaloMLP):
    """HQ-FSDP MLP whose weight "gathers" move no bytes.

    Every rank quantizes its rows of (WH)_Q under the shared scale into a
    CUDA-IPC buffer; the GEMMs (F: B operand split along N; E: operand split
    along its contracted dim) read the peers' rows in place over NVLink
    (halo_linear_set_qweight_sharded).  The absmax all-reduce of
    hqfsdp.hpp:172-196 and the ordering of shard writes before peer reads are
    one stream-ordered mailbox kernel each (halo_peer_sync); the backward
    regather (:243-266) is free because the forward's codes stay resident
    under the saved scale.  The next step's first mailbox barrier also
    guarantees no peer still reads a shard when it is re-quantized.  The
    weight-gradient reduce-scatter (:271-300) is fused into the G GEMMs: each
    rank's epilogue TMA-stores its fp32 partial rows into the owning rank's
    receive slot over NVLink, and after one mailbox barrier the owner takes
    the rank-order double mean -- the reference's arithmetic, bit for bit.
    Needs out_features % (world * 256) == 0 for every projection.

    staged=True bounds the NVLink bytes: right after the "shards written"
    barrier every rank copies each peer's shard once into a local gathered
    buffer (copy engine, cudaMemcpyAsync over the IPC mapping) and the GEMMs
    read that local copy -- (world-1)/world * n*m code bytes per weight and
    step cross NVLink, independent of the GEMM's tile raster (the in-place
    reads fetch a B panel once per M-tile unless it hits in L2).  Results are
    bit-identical either way (the same codes feed the same GEMMs).
    """

    def __init__(self, w_gate, w_up, w_down, scheme, group=None, check_stale=False, grad_dtype=torch.bfloat16,
                 staged: bool = False):
        super().__init__(w_gate, w_up, w_down, scheme, group, check_stale, grad_dtype, data_plane=None,
                         overlap=False)
        self.staged = staged
        from ._lib import HALO_OK  # noqa: F401  (library loaded)
        for p in self.params:
            if p.pad_rows or p.shard_rows % 256:
                raise ValueError("PeerFsdpHaloMLP: out_features must be a multiple of world * 256")
        self.buffers = []  # no gathered copies
        code_dt = torch.int8 if self.fmt == INT8 else torch.uint8
        self.local = [PeerBuffer(p.shard_rows * p.cols) for p in self.params]
        self.local_views = [b.tensor((p.shard_rows, p.cols), code_dt) for b, p in zip(self.local, self.params)]
        self.mailbox = PeerBuffer(3 * self.world * 4)  # flags + two absmax banks (halo_peer_sync)
        dev = self.params[0].master.device
        self.amax = [torch.zeros(1, dtype=torch.float32, device=dev) for _ in self.params]
        self.scales = [torch.ones(1, dtype=torch.float32, device=dev) for _ in self.params]
        # receive buffers of the fused gradient reduce-scatter: [world][shard_rows][cols] fp32
        self.recv = [PeerBuffer(self.world * p.shard_rows * p.cols * 4) for p in self.params]
        handles = _exchange(([b.handle() for b in self.local], self.mailbox.handle(),
                             [b.handle() for b in self.recv]), group)
        self._opened = []
        self.parts = []
        for i in range(len(self.params)):
            row = []
            for j in range(self.world):
                if j == self.rank:
                    row.append(self.local[i].ptr)
                else:
                    ptr = _ipc_open(handles[j][0][i])
                    self._opened.append(ptr)
                    row.append(ptr)
            self.parts.append(row)
        self.boxes = []
        for j in range(self.world):
            if j == self.rank:
                self.boxes.append(self.mailbox.ptr)
            else:
                ptr = _ipc_open(handles[j][1])
                self._opened.append(ptr)
                self.boxes.append(ptr)
        self.recv_parts = []
        for i in range(len(self.params)):
            row = []
            for j in range(self.world):
                if j == self.rank:
                    row.append(self.recv[i].ptr)
                else:
                    ptr = _ipc_open(handles[j][2][i])
                    self._opened.append(ptr)
                    row.append(ptr)
            self.recv_parts.append(row)
        self.epoch = 0
        self.staging = []
        if staged:
            self.staging = [torch.empty((p.shard_rows * self.world, p.cols), dtype=code_dt, device=dev)
                            for p in self.params]
        for i, (layer, parts, scale, recv) in enumerate(zip(self.layers, self.parts, self.scales, self.recv_parts)):
            if staged:
                layer.set_qweight(self.staging[i], scale)
            else:
                layer.set_qweight_sharded(parts, scale, keepalive=self)
            layer.set_grad_scatter(recv, self.rank)

    def _stage(self):
        """Copy every peer's shard into the local gathered buffers (NVLink,
        copy engine), stream-ordered after the shards-written barrier."""
        import ctypes as C
        from . import halo
        from ._lib import check, lib
        for i, p in enumerate(self.params):
            nb = p.shard_rows * p.cols
            base = self.staging[i].data_ptr()
            for j in range(self.world):
                check(lib().halo_device_copy(C.c_void_p(base + j * nb), C.c_void_p(self.parts[i][j]), nb,
                                             halo._stream()))

    def _sync(self, amax_in=None, amax_out=None):
        import ctypes as C
        from . import halo
        from ._lib import check, lib
        self.epoch += 1
        arr = (C.c_void_p * self.world)(*self.boxes)
        check(lib().halo_peer_sync(arr, self.world, self.rank, self.epoch, halo._ptr(amax_in), halo._ptr(amax_out),
                                   halo._stream()))

    def forward(self, x):
        import ctypes as C
        from . import halo
        from ._lib import check, lib
        ops = CudaOps()
        for i, p in enumerate(self.params):
            am = ops.absmax(p.master, self.block, self.rotate).reshape(1).float()
            # absmax "all-reduce": posted to every mailbox, max taken on device
            self._sync(am, self.amax[i])
            # quantize straight into the IPC-exported shard; the kernel derives
            # the shared scale from the exchanged absmax (compute_scales)
            check(lib().halo_rotate_quantize_amax(halo._ptr(p.master), halo._dt(p.master), p.shard_rows, p.cols,
                                                  self.block if self.rotate else -1, p.format,
                                                  halo._ptr(self.amax[i]), C.c_void_p(self.local[i].ptr),
                                                  halo._ptr(self.scales[i]), halo._stream()))
            p.global_scale = self.scales[i]
            p.local_absmax = am
            p.scales_valid = True
            self.ledger.record(self.ledger.scale_reduce, K_SCALE_BYTES, p.world)
            elems = p.shard_rows * p.world * p.cols
            self.ledger.record(self.ledger.gather, code_payload_bytes(p.format, elems) + K_SCALE_BYTES, p.world)
            self.ledger.bf16_gather_payload += 2 * elems
        self._sync()  # every rank's shards written before any peer GEMM reads them
        if self.staged:
            self._stage()
        return self.mlp.forward(x)

    def backward(self, dy):
        for p in self.params:
            if not p.scales_valid:
                raise HaloLogicError("backward_regather: no saved forward scales")
            self.ledger.backward_gathers += 1  # served in place: the codes never left
            self.ledger.backward_consumers += 1
        if self.check_stale:
            # backward_regather's stale check (hqfsdp.hpp:256-259): the codes
            # read in place were quantized under the forward's absmax; raise
            # if any rank's master shard changed since (flag max over ranks)
            ops = CudaOps()
            stale = torch.zeros(1, dtype=torch.float32, device=self.params[0].master.device)
            for p in self.params:
                am = ops.absmax(p.master, self.block, self.rotate).reshape(1).float()
                stale = torch.maximum(stale, (am != p.local_absmax.reshape(1).float()).float())
            if dist.is_initialized() and dist.get_world_size(self.group) > 1:
                dist.all_reduce(stale, op=dist.ReduceOp.MAX, group=self.group)
            if float(stale.item()) != 0.0:
                raise HaloLogicError("backward_regather: saved scales are stale (weights changed since the forward)")
        # G GEMMs stored every rank's fp32 partial rows into their owners'
        # receive slots; once all ranks are past them, each owner takes the
        # rank-order double mean of its rows (hqfsdp.hpp:288-292)
        dx, _ = self.mlp.backward(dy)
        self._sync()
        import ctypes as C
        from . import halo
        from ._lib import check, lib
        shards = []
        for i, p in enumerate(self.params):
            g = torch.empty((p.shard_rows, p.cols), dtype=self.layers[i].grad_dtype, device=p.master.device)
            check(lib().halo_reduce_scatter_shard(C.c_void_p(self.recv[i].ptr), self.world, p.shard_rows, p.cols,
                                                  halo._ptr(g), halo._dt(g), halo._stream()))
            self.ledger.record(self.ledger.reduce_scatter, 2 * p.shard_rows * p.world * p.cols, p.world)
            shards.append(g)
        return dx, shards

    def close(self):
        from ._lib import lib
        torch.cuda.synchronize()
        for layer in self.layers:
            layer.set_qweight_sharded(None, None)
            layer.set_grad_scatter(None, 0)
        for ptr in self._opened:
            lib().halo_ipc_close(ptr)
        self._opened = []
        for b in self.local + self.recv + [self.mailbox]:
            b.free()
