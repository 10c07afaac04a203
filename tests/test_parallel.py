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


# ---------------------------------------------------------------------------
# Row parallel (K-sharded; SURVEY.md 8e "K", 8f row f3): gloo world_size 2
# with the oracle as each rank's compute, and the column -> row MLP pairing
# ---------------------------------------------------------------------------
def _oracle_row_ops(wc_shard, ws, b, n0=N0, bits=4):
    """The three local steps of RowParallelLinear on the oracle."""
    qmax = (1 << (bits - 1)) - 1

    def local_amax(xs):
        y = O.group_rotate(xs.numpy(), O.ROT_REGULAR, n0)
        return torch.from_numpy(np.abs(y).max(axis=1) if y.shape[1] else np.zeros(y.shape[0]))

    def local_partial(xs, amax):
        y = O.group_rotate(xs.numpy(), O.ROT_REGULAR, n0)
        a = amax.numpy()
        s = np.where(a == 0.0, 1.0, a / qmax)  # compute_scales, quant.cpp:21
        codes = O.quantize(y, s, bits)
        return torch.from_numpy(O.int_gemm(codes, wc_shard, bits, bits)), torch.from_numpy(s)

    def deq(acc, s):
        return torch.from_numpy(O.dequant(acc.numpy(), s.numpy(), ws, b))

    return local_amax, local_partial, deq


def _row_worker(rank, world, port, q):
    from paper_2512_03673_b200.parallel import RowParallelLinear
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, w, b = _inputs()
        wc, ws = O.prepare_layer(w, O.ROT_REGULAR, N0)       # full-K scales
        lo, hi = shard_range(K, rank, world)
        layer = RowParallelLinear(K, N, *_oracle_row_ops(wc[:, lo:hi], ws, b))
        out = {"row": layer(torch.from_numpy(np.ascontiguousarray(x[:, lo:hi]))).numpy()}
        # MLP pair: fc1 column-parallel (no gather) feeds fc2 row-parallel
        w2 = O.from_bf16_bits(O.synth_input(N // 2, N, "gaussian", 8))
        wc2, ws2 = O.prepare_layer(w2, O.ROT_REGULAR, 4)
        c0, c1 = shard_range(N, rank, world)
        w1c, w1s = O.prepare_layer(w[c0:c1], O.ROT_REGULAR, N0)
        fc1 = ColumnParallelLinear(N, lambda xt: torch.from_numpy(
            O.forward(xt.numpy(), w1c, w1s, b[c0:c1], O.ROT_REGULAR, N0)["values"]))
        h = fc1(torch.from_numpy(x), gather=False)              # [M, N/P] = fc2's K shard
        fc2 = RowParallelLinear(N, N // 2, *_oracle_row_ops(wc2[:, c0:c1], ws2, None, n0=4))
        out["mlp"] = fc2(h).numpy()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_row_parallel_gloo_world2_bit_exact():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_row_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, w, b = _inputs()
    wc, ws = O.prepare_layer(w, O.ROT_REGULAR, N0)
    full = O.forward(x, wc, ws, b, O.ROT_REGULAR, N0)["values"]
    w2 = O.from_bf16_bits(O.synth_input(N // 2, N, "gaussian", 8))
    wc2, ws2 = O.prepare_layer(w2, O.ROT_REGULAR, 4)
    mlp = O.forward(full, wc2, ws2, None, O.ROT_REGULAR, 4)["values"]
    for r in range(world):
        assert np.array_equal(results[r]["row"], full)
        assert np.array_equal(results[r]["mlp"], mlp)


def test_row_parallel_capacity_precheck():
    from paper_2512_03673_b200._abi import CapacityError
    from paper_2512_03673_b200.parallel import RowParallelLinear
    with pytest.raises(CapacityError):  # int8: K <= 133,144 (pipeline.cpp:184-192)
        RowParallelLinear(200_000, 8, None, None, None, bits=(8, 8))


@pytest.mark.gpu
@pytest.mark.parametrize("P,bits,n0", [(2, 4, 16), (4, 4, 16), (3, 4, 4), (2, 8, 16)])
def test_row_shards_on_gpu_match_full_layer(P, bits, n0):
    """K-shards through the sm_100a kernels on one device: global max from the
    shards' exact maxima, per-shard K1 + int32 partial GEMM, summed, dequant --
    equal to the unsharded forward (i32 / f32 / bf16), codes = the full
    codes' columns."""
    import paper_2512_03673_b200 as crt
    from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec
    from paper_2512_03673_b200.analysis import rotated_row_absmax
    dev = "cuda"
    m, k, n = 300, 3072, 768
    to_t = lambda bits_: torch.from_numpy(bits_.astype(np.uint16).view(np.int16)).to(dev).view(torch.bfloat16)  # noqa: E731
    x, w = to_t(O.synth_input(m, k, "rowwise", 21)), to_t(O.synth_input(n, k, "gaussian", 22))
    bias = torch.randn(n, device=dev)
    spec, q = RotationSpec(RotationKind.regular, n0), QuantSpec(bits)
    full = crt.prepare_layer(w, bias, spec, q)
    ks = k // P
    shards = [crt.prepare_layer_kshard(w, bias, spec, q, r, P) for r in range(P)]
    assert all((s.out_features, s.in_features) == (n, ks) for s in shards)
    xs = [x[:, r * ks:(r + 1) * ks].contiguous() for r in range(P)]
    amax = torch.stack([rotated_row_absmax(t, spec) for t in xs]).max(0).values.contiguous()
    i8 = bits == 4
    parts = [crt.rotate_quantize_amax(t, spec, amax, int8_codes=i8, bits=bits) for t in xs]
    codes_full, s_full = crt.rotate_quantize(x, spec, q)
    for r, (c, s32, sums) in enumerate(parts):
        assert torch.equal(s32, s_full)
        if i8:
            got = c[:, :ks].view(torch.int8).to(torch.int32)
            pf = codes_full[:, :k // 2].to(torch.int32)
            lo = torch.where((pf & 15) >= 8, (pf & 15) - 16, pf & 15)
            hi = torch.where((pf >> 4) >= 8, (pf >> 4) - 16, pf >> 4)
            want = torch.stack([lo, hi], 2).reshape(m, k)[:, r * ks:(r + 1) * ks]
            assert torch.equal(got, want)
            assert torch.equal(sums, want.sum(1).to(torch.int32))
    if i8:
        acc = sum(crt.quant_gemm_i8(c, s, su, L, out="i32") for (c, s, su), L in zip(parts, shards))
    else:
        acc = sum(crt.quant_gemm(c, s, L, q, out="i32") for (c, s, _), L in zip(parts, shards))
    acc = acc.to(torch.int32).contiguous()
    assert torch.equal(acc, crt.forward(x, full, q, out="i32"))
    for out in ("f32", "bf16", "i32"):
        assert torch.equal(crt.dequant(acc, s_full, shards[0], out=out),
                           crt.forward(x, full, q, out=out)), out


@pytest.mark.gpu
def test_kshard_rejects_straddling_groups():
    import paper_2512_03673_b200 as crt
    from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec, ShapeError
    w = torch.randn(64, 96, device="cuda").to(torch.bfloat16)
    with pytest.raises(ShapeError):  # 96/2 = 48 not a multiple of 64
        crt.prepare_layer_kshard(w, None, RotationSpec(RotationKind.regular, 64), QuantSpec(4), 0, 2)
    with pytest.raises(ShapeError):  # 96 % 5 != 0
        crt.prepare_layer_kshard(w, None, RotationSpec(RotationKind.regular, 4), QuantSpec(4), 0, 5)
