"""Tensor parallelism through the C-ABI (crt_nccl_*, crt_tp_layer_prepare,
crt_tp_forward; SURVEY.md 8(b) "Multi-GPU", 8(e)).

CPU: the entry points exist, NCCL resolves, and argument errors come back
synchronously with the reference taxonomy (+ CRT_ERR_NCCL).
GPU, one device: a 1-rank NCCL communicator runs the whole collective path
(all-gather + interleave, MAX / SUM all-reduces) and must equal the plain
forward bit for bit.  GPU, two devices (skipped on one): two processes,
column-parallel fc1 without gather feeding row-parallel fc2, against the
single-GPU forward."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch

import paper_2512_03673_b200 as crt
from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec, _abi


def test_nccl_unique_id_and_errors_cpu():
    lib = _abi.load()
    uid = (ctypes.c_uint8 * 128)()
    st = lib.crt_nccl_unique_id(uid)
    if st == _abi.CRT_ERR_NCCL:
        pytest.skip("libnccl.so.2 not loadable here")
    assert st == _abi.CRT_OK and any(bytes(uid))
    r, n = ctypes.c_int32(), ctypes.c_int32()
    assert lib.crt_nccl_comm_info(None, ctypes.byref(r), ctypes.byref(n)) == _abi.CRT_ERR_INVALID_VALUE
    desc = _abi.LayerDescC(8, 16, RotationSpec(RotationKind.regular, 16).c(), 4, 0)
    h = ctypes.c_void_p()
    assert lib.crt_tp_layer_prepare(ctypes.byref(desc), None, 16, None, 1, None, None,
                                    ctypes.byref(h)) == _abi.CRT_ERR_INVALID_VALUE
    assert lib.crt_tp_layer_prepare(ctypes.byref(desc), None, 16, None, 7, None, None,
                                    ctypes.byref(h)) == _abi.CRT_ERR_INVALID_VALUE
    assert lib.crt_tp_forward(None, None, 0, 1, 16, 0, None, 8, 1, None, None, None) == \
        _abi.CRT_ERR_INVALID_VALUE
    assert lib.crt_nccl_comm_create(2, 2, uid, ctypes.byref(h)) == _abi.CRT_ERR_INVALID_VALUE
    with pytest.raises(crt.Error):
        _abi.check(_abi.CRT_ERR_NCCL)


def _data(M, K, N, seed, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    x = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    w = torch.randn(N, K, device=dev, generator=g).to(torch.bfloat16)
    b = torch.randn(N, device=dev, generator=g)
    return x, w, b


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("out", ["bf16", "f32", "i32"])
def test_single_rank_tp_equals_forward(bits, out):
    from paper_2512_03673_b200.parallel import NcclComm, TensorParallelLinear
    dev = torch.device("cuda", 0)
    spec = RotationSpec(RotationKind.regular, 16)
    q = QuantSpec(bits)
    comm = NcclComm()
    assert (comm.rank, comm.nranks) == (0, 1)
    for (M, K, N) in [(300, 1024, 768), (129, 3072, 2048)]:
        x, w, b = _data(M, K, N, 11 + bits + M, dev)
        ref = crt.forward(x, crt.prepare_layer(w, b, spec, q), q, out=out)
        col = TensorParallelLinear(w, b, spec, q, q, "column", comm)
        row = TensorParallelLinear(w, b, spec, q, q, "row", comm)
        yc = col(x, gather=True, out=out)
        yr = row(x, out=out)
        torch.cuda.synchronize()
        assert torch.equal(yc, ref) and torch.equal(yr, ref), (M, K, N)
    comm.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _two_rank_worker(rank, port, q):
    import torch.distributed as dist

    from paper_2512_03673_b200.parallel import NcclComm, TensorParallelLinear
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    spec = RotationSpec(RotationKind.regular, 16)
    q4 = QuantSpec(4)
    M, D, F = 256, 1024, 4096
    x, w1, b1 = _data(M, D, F, 5, dev)
    _, w2, b2 = _data(M, F, D, 6, dev)
    want = crt.forward(crt.forward(x, crt.prepare_layer(w1, b1, spec)),
                       crt.prepare_layer(w2, b2, spec))
    comm = NcclComm()
    fc1 = TensorParallelLinear(w1, b1, spec, q4, q4, "column", comm)
    fc2 = TensorParallelLinear(w2, b2, spec, q4, q4, "row", comm)
    got = fc2(fc1(x, gather=False))
    gath = fc1(x, gather=True)
    torch.cuda.synchronize()
    ok = torch.equal(got, want) and torch.equal(
        gath, crt.forward(x, crt.prepare_layer(w1, b1, spec)))
    q.put((rank, bool(ok)))
    comm.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_two_rank_colrow_mlp_bit_identical():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_two_rank_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


@pytest.mark.gpu
def test_forward_rejects_bad_output_buffers():
    dev = torch.device("cuda", 0)
    spec = RotationSpec(RotationKind.regular, 16)
    x, w, b = _data(64, 256, 128, 3, dev)
    layer = crt.prepare_layer(w, b, spec)
    with pytest.raises(crt.InvalidValueError):  # f32 into a bf16 buffer
        crt.forward(x, layer, out="f32", y=torch.empty(64, 128, dtype=torch.bfloat16, device=dev))
    with pytest.raises(crt.ShapeError):  # too few rows
        crt.forward(x, layer, y=torch.empty(32, 128, dtype=torch.bfloat16, device=dev))
    with pytest.raises(crt.ShapeError):  # strided columns
        crt.forward(x, layer, y=torch.empty(64, 256, dtype=torch.bfloat16, device=dev)[:, ::2])
    xn = x.clone()
    xn[5, 7] = float("nan")
    with pytest.raises(crt.InvalidValueError):  # the reference throws (quant.cpp:16-18)
        crt.forward(xn, layer)
    crt.forward(x, layer)  # a fresh call on the same default workspace is clean
    ws = crt.Workspace(64, 256, dev)
    crt.forward(xn, layer, workspace=ws, check_finite=False)
    crt.forward(x, layer)  # another workspace's word is not this one's
    with pytest.raises(crt.InvalidValueError):
        ws.status()
    ws.status()  # cleared
    wn = w.clone()
    wn[3, 3] = float("inf")
    with pytest.raises(crt.InvalidValueError):  # compute_scales on the weights
        crt.prepare_layer(wn, b, spec)
