"""Multi-GPU sharding of the ConvLinear4bit path.

One process per GPU; torch.distributed (NCCL over NVLink/NVSwitch) is the
plumbing.  Two strategies, both bit-identical to one GPU:

* Column parallel (wide layers, e.g. FLUX fc1 N = 12288): rank r owns output
  channels [r*N/P, (r+1)*N/P).  Its weight shard is prepared from those rows
  of W (``crt_layer_prepare_shard``), so codes / scales / bias are exactly the
  full layer's rows; X is replicated and every rank runs K1 itself (per-token
  scales span the full K exactly like the reference), then K3 on its shard.
  The shards are reassembled with one ``all_gather_into_tensor`` (rank-major
  [P][M][N/P]) and a column interleave into [M, N].
* Row parallel (SURVEY.md 8e "K", 8f row f3; e.g. FLUX fc2 K = 12288, fed by
  the column-parallel fc1 whose output shard IS this rank's input shard):
  rank r owns input columns [r*K/P, (r+1)*K/P) of the full layer's codes
  (``crt_layer_prepare_kshard``: per-channel scales over all of K).  Each
  rank computes the exact max |group_rotate(x)| of its columns, one MAX
  all-reduce (M doubles) gives the global per-token max, so K1 produces
  exactly the unsharded scales and codes on its columns; K3 yields int32
  partial accumulators and one SUM all-reduce (int32: exact, order-free)
  gives int_gemm's result, dequantised once (``crt_dequant``).
* Prompt (batch) sharding: independent prompts go to ranks round-robin; no
  collective on the data path.

The local compute is injectable (``local_forward``) so the host logic --
shard ranges, the collective, the reassembly -- is testable on CPU with the
``gloo`` backend and the oracle standing in for the GPU kernels
(tests/test_parallel.py).  The product path uses the CUDA kernels only.

``TensorParallelLinear`` is the same two strategies through the C-ABI's
tensor-parallel entry points (crt_tp_layer_prepare / crt_tp_forward): the
NCCL collectives, the all-gather interleave and the row-parallel max / sum
all-reduces run inside the library on one NCCL communicator
(``NcclComm``), so a C++ host gets the identical sharded path.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, nranks: int) -> Tuple[int, int]:
    """[begin, end) of the output channels owned by `rank` (N % P == 0, as
    crt_layer_prepare_shard requires)."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("bad rank / nranks")
    if n % nranks:
        raise ValueError(f"out_features {n} not divisible by {nranks} ranks")
    step = n // nranks
    return rank * step, (rank + 1) * step


def prompt_shard(n_prompts: int, rank: int, nranks: int) -> List[int]:
    """Prompt indices processed by `rank` (round-robin, no communication)."""
    return list(range(rank, n_prompts, nranks))


def interleave_rank_major(gathered: torch.Tensor, nranks: int) -> torch.Tensor:
    """[P*M, N/P] rank-major all-gather output -> [M, N] (rank r's columns at
    [r*N/P, (r+1)*N/P))."""
    pm, ns = gathered.shape
    m = pm // nranks
    return gathered.view(nranks, m, ns).permute(1, 0, 2).reshape(m, nranks * ns)


class ColumnParallelLinear:
    """A ConvLinear4bit layer sharded over output channels.

    ``local_forward(x) -> y_shard [M, N/P]`` computes this rank's columns;
    by default it is the CUDA path on a layer prepared with
    ``prepare_layer_shard``.  ``forward`` all-gathers the shards."""

    def __init__(self, out_features: int, local_forward: Callable[[torch.Tensor], torch.Tensor],
                 group: Optional[dist.ProcessGroup] = None):
        self.group = group
        self.nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.out_features = out_features
        self.cols = shard_range(out_features, self.rank, self.nranks)
        self.local_forward = local_forward

    @classmethod
    def from_weights(cls, w: torch.Tensor, bias: Optional[torch.Tensor], rotation, wq,
                     aq, out: str = "bf16", group: Optional[dist.ProcessGroup] = None,
                     name: str = ""):
        """CUDA path: prepare this rank's shard with the sm_100a kernels."""
        from . import api
        nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        layer = api.prepare_layer_shard(w, bias, rotation, wq, rank, nranks, name)

        def local_forward(x):
            return api.forward(x, layer, aq, out=out)

        obj = cls(w.shape[0], local_forward, group)
        obj.layer = layer
        return obj

    def forward(self, x: torch.Tensor, gather: bool = True) -> torch.Tensor:
        """gather=False returns this rank's [M, N/P] shard -- the input shard
        of a following RowParallelLinear (no collective between them)."""
        shard = self.local_forward(x).contiguous()
        if self.nranks == 1 or not gather:
            return shard
        gathered = torch.empty((self.nranks * shard.shape[0], shard.shape[1]), dtype=shard.dtype,
                               device=shard.device)
        dist.all_gather_into_tensor(gathered, shard, group=self.group)
        return interleave_rank_major(gathered, self.nranks)

    __call__ = forward


INT32_MAX = 2147483647


class RowParallelLinear:
    """A ConvLinear4bit layer sharded over input features.

    ``forward(x_shard)`` takes this rank's [M, K/P] input columns and returns
    the full [M, N] output on every rank, equal to the unsharded forward bit
    for bit.  The local steps are injectable (CPU tests use the oracle):
      local_amax(x_shard) -> float64 [M]: exact max |group_rotate| of the shard
      local_partial(x_shard, amax) -> (int32 [M, N] partial acc, fp32/f64 [M] scales)
      dequant(acc, scales) -> y
    """

    def __init__(self, in_features: int, out_features: int, local_amax, local_partial, dequant,
                 bits: Tuple[int, int] = (4, 4), group: Optional[dist.ProcessGroup] = None):
        self.group = group
        self.nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.in_features, self.out_features = in_features, out_features
        self.cols = shard_range(in_features, self.rank, self.nranks)
        qa, qw = (1 << (bits[0] - 1)) - 1, (1 << (bits[1] - 1)) - 1
        if qa * qw * in_features > INT32_MAX:  # int_gemm capacity, pipeline.cpp:184-192
            from ._abi import CapacityError
            raise CapacityError(f"int_gemm: {in_features}-deep accumulation can overflow int32")
        self.local_amax, self.local_partial, self.dequant = local_amax, local_partial, dequant

    @classmethod
    def from_weights(cls, w: torch.Tensor, bias: Optional[torch.Tensor], rotation, wq, aq,
                     out: str = "bf16", group: Optional[dist.ProcessGroup] = None,
                     name: str = ""):
        """CUDA path: this rank's K-shard prepared with the sm_100a kernels."""
        from . import api
        from .analysis import rotated_row_absmax
        nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        layer = api.prepare_layer_kshard(w, bias, rotation, wq, rank, nranks, name)
        i8 = aq.bits == 4 and wq.bits == 4

        def local_amax(xs):
            return rotated_row_absmax(xs, rotation)

        def local_partial(xs, amax):
            codes, s32, sums = api.rotate_quantize_amax(xs, rotation, amax, int8_codes=i8,
                                                        bits=aq.bits)
            if i8:
                acc = api.quant_gemm_i8(codes, s32, sums, layer, out="i32")
            else:
                acc = api.quant_gemm(codes, s32, layer, aq, out="i32")
            return acc, s32

        def deq(acc, s32):
            return api.dequant(acc, s32, layer, out=out)

        obj = cls(w.shape[1], w.shape[0], local_amax, local_partial, deq, (aq.bits, wq.bits),
                  group)
        obj.layer = layer
        return obj

    def forward(self, x_shard: torch.Tensor) -> torch.Tensor:
        amax = self.local_amax(x_shard).contiguous()
        if self.nranks > 1:
            dist.all_reduce(amax, op=dist.ReduceOp.MAX, group=self.group)
        acc, scales = self.local_partial(x_shard, amax)
        acc = acc.contiguous()
        if self.nranks > 1:
            dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=self.group)
        return self.dequant(acc, scales)

    __call__ = forward


def run_prompts(prompts: Sequence[torch.Tensor], fn: Callable[[torch.Tensor], torch.Tensor],
                group: Optional[dist.ProcessGroup] = None) -> List[Tuple[int, torch.Tensor]]:
    """Prompt sharding: this rank runs `fn` on its prompts; returns
    (prompt index, output) pairs.  No collective."""
    nranks = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    return [(i, fn(prompts[i])) for i in prompt_shard(len(prompts), rank, nranks)]


# ---------------------------------------------------------------------------
# The C-ABI tensor-parallel path (include/crt/convlinear4bit.h, crt_tp_*)
# ---------------------------------------------------------------------------
class NcclComm:
    """An NCCL communicator for the library's tensor-parallel entry points,
    one per rank on the current CUDA device.  The 128-byte unique id is made
    on rank 0 and broadcast over the torch.distributed group (any backend)."""

    def __init__(self, group: Optional[dist.ProcessGroup] = None):
        import ctypes

        from . import _abi
        self._abi = _abi
        lib = _abi.load()
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        uid = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            _abi.check(lib.crt_nccl_unique_id(uid))
        if self.nranks > 1:
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                       group=group)
            uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        _abi.check(lib.crt_nccl_comm_create(self.nranks, self.rank, uid, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._abi.load().crt_nccl_comm_destroy(self._h)
        self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class TensorParallelLinear:
    """A ConvLinear4bit layer sharded over the ranks of an ``NcclComm``
    through the C-ABI: ``mode="column"`` (output channels; x is the full
    input, ``forward(x, gather=False)`` returns the [M, N/P] shard) or
    ``mode="row"`` (input features; x is the rank's [M, K/P] columns, the
    output the full [M, N] on every rank).  Bit-identical to one GPU."""

    MODES = {"column": 1, "row": 2}

    def __init__(self, w: torch.Tensor, bias: Optional[torch.Tensor], rotation, wq, aq,
                 mode: str, comm: NcclComm, name: str = ""):
        import ctypes

        from . import _abi, api
        if mode not in self.MODES:
            raise ValueError("mode must be 'column' or 'row'")
        self.mode, self.comm, self.aq, self.name = mode, comm, aq, name
        self.nranks, self.rank = comm.nranks, comm.rank
        N, K = w.shape
        self.out_full, self.in_full = N, K
        if bias is not None:
            bias = bias.to(device=w.device, dtype=torch.float32).contiguous()
        desc = _abi.LayerDescC(N, K, rotation.c(), wq.bits, api._dtype_code(w))
        h = ctypes.c_void_p()
        with torch.cuda.device(w.device):
            _abi.check(_abi.load().crt_tp_layer_prepare(
                ctypes.byref(desc), api._ptr(w), w.stride(0), api._ptr(bias), self.MODES[mode],
                comm.handle, api._stream(w), ctypes.byref(h)))
        n_local = N // self.nranks if mode == "column" else N
        k_local = K // self.nranks if mode == "row" else K
        self.layer = api.PreparedLayer(h.value, n_local, k_local, rotation, wq, bias is not None,
                                       name, w.device, (self.rank, self.nranks))

    def forward(self, x: torch.Tensor, gather: bool = True, out: str = "bf16",
                y: Optional[torch.Tensor] = None, workspace=None) -> torch.Tensor:
        from . import _abi, api
        M, K = x.shape
        if K != self.layer.in_features:
            raise api.ShapeError(f"input has {K} columns, the shard expects {self.layer.in_features}")
        N = self.out_full if (self.mode == "row" or gather) else self.layer.out_features
        if y is None:
            y = torch.empty((M, N), dtype=api._OUT_DTYPE[out], device=x.device)
        else:
            api._check_out(y, M, N, out, self.layer.device)
        ws = workspace or api._workspace_for(M, K, x.device)
        _abi.check(_abi.load().crt_tp_forward(
            self.layer.handle, api._ptr(x), api._dtype_code(x), M, x.stride(0), api._OUT[out],
            api._ptr(y), y.stride(0), int(gather), ws.handle, self.comm.handle, api._stream(x)))
        return y

    __call__ = forward
