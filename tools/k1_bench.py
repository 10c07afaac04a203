"""Device-only K1 timing: back-to-back launches captured in a CUDA graph,
cycling over enough input buffers that every launch reads its input from
HBM (the set is > 2x the 126 MB L2), so host/launch overhead and L2 reuse
are both excluded.  Reports us per launch and GB/s on SURVEY 8(d)'s packed
algorithmic bytes (2 B in + 0.5 B codes per element + 4 B scale per row),
and on the bytes the int8-code layout actually moves (2 + 1 B + 8 B/row).

python tools/k1_bench.py [M K N0 bits] ...   (default: the FLUX shapes)
"""
import ctypes
import gc
import json
import sys

import torch

sys.path.insert(0, __import__("os").environ.get("CRT_ROOT", "."))
import paper_2512_03673_b200 as crt  # noqa: E402
from paper_2512_03673_b200 import RotationKind, RotationSpec  # noqa: E402
from paper_2512_03673_b200.api import _lib, check  # noqa: E402

L2 = 126 * 1024 * 1024


def k1_time(M, K, n0, bits=5, reps=6):
    spec = RotationSpec(RotationKind.regular if n0 > 1 else RotationKind.none, max(n0, 1))
    nbuf = max(2, -(-3 * L2 // (M * K * 2)))
    g = torch.Generator(device="cuda").manual_seed(1)
    xs = [torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16) for _ in range(nbuf)]
    ld = max(16, (K + 15) // 16 * 16) if bits != 4 else max(16, ((K + 1) // 2 + 15) // 16 * 16)
    codes = [torch.empty((M, ld), dtype=torch.uint8, device="cuda") for _ in range(nbuf)]
    s32 = [torch.empty(M, dtype=torch.float32, device="cuda") for _ in range(nbuf)]
    sums = [torch.empty(M, dtype=torch.int32, device="cuda") for _ in range(nbuf)]
    rc = spec.c()
    lib = _lib()
    st = torch.cuda.Stream()

    def launch(i):
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        if bits == 5:
            check(lib.crt_rotate_quant_i8(ctypes.c_void_p(xs[i].data_ptr()), 0, M, K, K,
                                          ctypes.byref(rc), ctypes.c_void_p(codes[i].data_ptr()),
                                          ld, ctypes.c_void_p(s32[i].data_ptr()),
                                          ctypes.c_void_p(sums[i].data_ptr()), s))
        else:
            check(lib.crt_rotate_quant(ctypes.c_void_p(xs[i].data_ptr()), 0, M, K, K,
                                       ctypes.byref(rc), bits,
                                       ctypes.c_void_p(codes[i].data_ptr()), ld,
                                       ctypes.c_void_p(s32[i].data_ptr()), None, s))

    with torch.cuda.stream(st):
        for i in range(nbuf):
            launch(i)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        for _ in range(reps):
            for i in range(nbuf):
                launch(i)
    n = reps * nbuf
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / n)
    us = sorted(ts)[len(ts) // 2]
    # release this graph and its buffers now: a second capture of the same
    # shape while they linger ran 10-25x slower (graph replays only; eager
    # launches are unaffected)
    del graph, xs, codes, s32, sums
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    packed = M * K * 2.5 + 4 * M
    moved = M * K * (3 if bits != 4 else 2.5) + (8 if bits == 5 else 4) * M
    return {"M": M, "K": K, "n0": n0, "bits": bits, "us": round(us, 2),
            "GBps_packed": round(packed / us / 1e3, 1), "GBps_moved": round(moved / us / 1e3, 1),
            "launches": n, "buffers": nbuf}


if __name__ == "__main__":
    args = sys.argv[1:]
    cases = []
    if args:
        for i in range(0, len(args), 4):
            cases.append(tuple(int(v) for v in args[i:i + 4]))
    else:
        cases = [(4608, 3072, 16, 5), (4608, 12288, 16, 5), (4096, 3072, 16, 5),
                 (4608, 3072, 16, 4), (4608, 12288, 16, 4),
                 (4608, 3072, 4, 5), (4608, 3072, 64, 5), (4608, 3072, 256, 5),
                 (4608, 15360, 16, 5), (512, 3072, 16, 5)]
    for c in cases:
        print(json.dumps(k1_time(*c)), flush=True)
