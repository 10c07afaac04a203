"""Multi-GPU sharding logic (paper_2512_03673_b200/parallel.py).

CPU: world_size-2 process groups on the gloo backend, with the oracle (the
plain-C restatement of the reference) standing in for each rank's GPU
compute -- proves that column-parallel sharding + all-gather + interleave
reproduces the full layer bit for bit (codes, accumulators and dequantised
values), and that prompt sharding covers every prompt once.
GPU: the same sharding through the sm_100a kernels on one device (the two
shards computed one after the other and interleaved like the all-gather).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2512_03673_b200.parallel import (ColumnParallelLinear, interleave_rank_major,
                                            prompt_shard, run_prompts, shard_range)


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_ranges_partition_the_channels():
    for n, p in [(12288, 8), (3072, 2), (3072, 4), (8, 8)]:
        ranges = [shard_range(n, r, p) for r in range(p)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    with pytest.raises(ValueError):
        shard_range(10, 0, 4)


def test_prompt_shard_covers_each_prompt_once():
    for n, p in [(8, 2), (8, 8), (8, 3), (1, 4)]:
        got = sorted(i for r in range(p) for i in prompt_shard(n, r, p))
        assert got == list(range(n))


def test_interleave_rank_major():
    m, p, ns = 3, 4, 2
    full = torch.arange(m * p * ns).view(m, p * ns)
    shards = [full[:, r * ns:(r + 1) * ns] for r in range(p)]
    gathered = torch.cat(shards, 0)  # what all_gather_into_tensor produces
    assert torch.equal(interleave_rank_major(gathered, p), full)


# ---------------------------------------------------------------------------
# gloo, world_size 2
# ---------------------------------------------------------------------------
M, K, N, N0 = 12, 256, 16, 16


def _inputs():
    x = O.from_bf16_bits(O.synth_input(M, K, "colwise", 5))
    w = O.from_bf16_bits(O.synth_input(N, K, "gaussian", 6))
    b = O.from_bf16_bits(O.to_bf16_bits(O.gaussian_matrix(1, N, 7)[0]))
    return x, w, b


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, w, b = _inputs()
        lo, hi = shard_range(N, rank, world)
        wc, ws = O.prepare_layer(w[lo:hi], O.ROT_REGULAR, N0)

        def local(xt, field):
            f = O.forward(xt.numpy(), wc, ws, b[lo:hi], O.ROT_REGULAR, N0)
            return torch.from_numpy(np.ascontiguousarray(f[field]))

        out = {}
        for field in ("values", "acc"):
            layer = ColumnParallelLinear(N, lambda xt, fl=field: local(xt, fl))
            out[field] = layer(torch.from_numpy(x)).numpy()
        # prompt sharding: 5 prompts, each rank its own, gathered for checking
        prompts = [torch.from_numpy(x[i:i + 2]) for i in range(5)]
        mine = run_prompts(prompts, lambda t: t.sum())
        allp = [None] * world
        dist.all_gather_object(allp, [i for i, _ in mine])
        out["prompts"] = sorted(i for lst in allp for i in lst)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_column_parallel_gloo_world2_bit_exact():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, w, b = _inputs()
    wc, ws = O.prepare_layer(w, O.ROT_REGULAR, N0)
    full = O.forward(x, wc, ws, b, O.ROT_REGULAR, N0)
    for r in range(world):
        assert np.array_equal(results[r]["acc"], full["acc"])
        assert np.array_equal(results[r]["values"], full["values"])
        assert results[r]["prompts"] == list(range(5))


# ---------------------------------------------------------------------------
# GPU: shards through the sm_100a kernels on one device
# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4])
def test_column_shards_on_gpu_match_full_layer(P):
    import paper_2512_03673_b200 as crt
    from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec
    dev = "cuda"
    m, k, n = 300, 3072, 768
    xb = O.synth_input(m, k, "rowwise", 11)
    wb = O.synth_input(n, k, "gaussian", 12)
    to_t = lambda bits: torch.from_numpy(bits.astype(np.uint16).view(np.int16)).to(dev).view(torch.bfloat16)  # noqa: E731
    x, w = to_t(xb), to_t(wb)
    bias = torch.randn(n, device=dev)
    spec = RotationSpec(RotationKind.regular, 16)
    full = crt.prepare_layer(w, bias, spec)
    shards = [crt.prepare_layer_shard(w, bias, spec, QuantSpec(4), r, P) for r in range(P)]
    for out in ("i32", "f32", "bf16"):
        ref = crt.forward(x, full, QuantSpec(4), out=out)
        parts = [crt.forward(x, s, QuantSpec(4), out=out) for s in shards]
        got = interleave_rank_major(torch.cat(parts, 0), P)
        assert torch.equal(got, ref), out
