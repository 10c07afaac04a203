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
* Prompt (batch) sharding: independent prompts go to ranks round-robin; no
  collective on the data path.

The local compute is injectable (``local_forward``) so the host logic --
shard ranges, the collective, the reassembly -- is testable on CPU with the
``gloo`` backend and the oracle standing in for the GPU kernels
(tests/test_parallel.py).  The product path uses the CUDA kernels only.
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

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        shard = self.local_forward(x).contiguous()
        if self.nranks == 1:
            return shard
        gathered = torch.empty((self.nranks * shard.shape[0], shard.shape[1]), dtype=shard.dtype,
                               device=shard.device)
        dist.all_gather_into_tensor(gathered, shard, group=self.group)
        return interleave_rank_major(gathered, self.nranks)

    __call__ = forward


def run_prompts(prompts: Sequence[torch.Tensor], fn: Callable[[torch.Tensor], torch.Tensor],
                group: Optional[dist.ProcessGroup] = None) -> List[Tuple[int, torch.Tensor]]:
    """Prompt sharding: this rank runs `fn` on its prompts; returns
    (prompt index, output) pairs.  No collective."""
    nranks = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    return [(i, fn(prompts[i])) for i in prompt_shard(len(prompts), rank, nranks)]
