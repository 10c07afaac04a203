#!/usr/bin/env python
"""bench.py -- W4A4 ConvLinear4bit forward at the FLUX.1-dev MLP shapes.

Workload (BASELINE.json configs[1], the largest single-GPU config the metric
is quoted on): one "step" is the FLUX.1-dev MLP pair through the
ConvLinear4bit path, N0 = 16, W4A4:
    fc1: x[4608, 3072]  -> K1 rotate+quant -> K3 GEMM vs W1[12288, 3072] -> y1 bf16
    fc2: y1[4608,12288] -> K1 rotate+quant -> K3 GEMM vs W2[3072, 12288] -> y2 bf16
value  = 2*M*N*K summed over both layers / device time of the step (TOPS),
         inputs resident in HBM, L2 flushed (256 MiB write) between steps.
e2e    = same metric through the public API with HOST buffers: pinned x ->
         device, both layers, y2 -> pinned host, every step.
N > 1  = independent replicas (batch-8 prompt sharding): every rank runs the
         full step on its own prompt; no data-path collective ("weak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "W4A4 ConvLinear4bit TOPS at FLUX.1 shapes; rot+quant HBM GB/s; vs CPU ref"
M_TOK, D_MODEL, D_FF, N0 = 4608, 3072, 12288, 16
WORKLOAD = ("FLUX.1-dev MLP pair: fc1 M=4608,K=3072,N=12288 and fc2 M=4608,K=12288,N=3072, "
            "N0=16, W4A4 (configs[1])")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n0", type=int, default=N0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=6.0,
                    help="--impl reference: CPU seconds per step (bounded sample of the rows)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras)")
    ap.add_argument("--path", choices=["v3", "v2"], default="v3",
                    help="K1+K3 pair: v3 (int8 activation codes -> K3 v4, or K3 v3 under "
                         "CRT_K3_V3=1; what forward() runs) or v2 (packed codes, "
                         "software expansion)")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config blocks (cfg1, cfg3 N0 sweep, cfg4 FLUX stack)")
    ap.add_argument("--cpu-stages", type=int, default=0, metavar="ROWS",
                    help=argparse.SUPPRESS)  # child process: staged CPU reference timing
    ap.add_argument("--parallel", choices=["replica", "column", "colrow"], default="replica",
                    help="N>1: independent prompt replicas (weak scaling, default); column: "
                         "fc1 and fc2 column-parallel, each output all-gathered (configs[4]); "
                         "colrow: fc1 column-parallel WITHOUT a gather feeding fc2 "
                         "row-parallel (one int32 SUM + M-double MAX all-reduce) -- both "
                         "through the C-ABI tensor-parallel path (crt_tp_*, NCCL), strong scaling")
    return ap.parse_args()


def layer_ops():
    return 2 * M_TOK * D_FF * D_MODEL + 2 * M_TOK * D_MODEL * D_FF


# ---------------------------------------------------------------------------
# CPU arm: the reference's own implementation (oracle/_ref, compiled from the
# unmodified reference sources) on a bounded row sample of the same workload.
# Rows are independent (per-token scales), so a row sample is the same work
# per row as the full step.
# ---------------------------------------------------------------------------
class CpuReference:
    def __init__(self, threads: int, seed: int = 0):
        os.environ["CONVROT_THREADS"] = str(threads)
        import numpy as np
        import oracle as O
        self.O = O
        self.np = np
        self.kind = "reference" if O.ref_available() else "port"
        self.threads = threads if self.kind == "reference" else 1
        rng = np.random.default_rng(seed)
        # bf16-representable synthetic data (same distribution as the GPU arm)
        def bf16(a):
            return O.from_bf16_bits(O.to_bf16_bits(a))
        self.w1 = bf16(rng.standard_normal((D_FF, D_MODEL)))
        self.w2 = bf16(rng.standard_normal((D_MODEL, D_FF)))
        self.b1 = bf16(rng.standard_normal(D_FF))
        self.b2 = bf16(rng.standard_normal(D_MODEL))
        self.x_all = bf16(rng.standard_normal((4096, D_MODEL)))
        if self.kind == "reference":
            self.l1 = O.Ref.prepare_layer(self.w1, self.b1, O.ROT_REGULAR, N0)
            self.l2 = O.Ref.prepare_layer(self.w2, self.b2, O.ROT_REGULAR, N0)
        else:
            self.l1 = O.prepare_layer(self.w1, O.ROT_REGULAR, N0)
            self.l2 = O.prepare_layer(self.w2, O.ROT_REGULAR, N0)

    def step(self, rows: int) -> float:
        O = self.O
        x = self.x_all[:rows]
        t0 = time.perf_counter()
        if self.kind == "reference":
            y1 = O.Ref.forward_prepared(x, self.l1[0], self.l1[1], self.b1, O.ROT_REGULAR, N0)
            O.Ref.forward_prepared(y1, self.l2[0], self.l2[1], self.b2, O.ROT_REGULAR, N0)
        else:
            y1 = O.forward(x, self.l1[0], self.l1[1], self.b1, O.ROT_REGULAR, N0)["values"]
            O.forward(y1, self.l2[0], self.l2[1], self.b2, O.ROT_REGULAR, N0)
        return time.perf_counter() - t0

    def calibrate(self, target_s: float = 12.0, max_rows: int = 4096) -> int:
        rows = 16
        t = self.step(rows)
        while t < target_s / 4 and rows < max_rows:
            rows = min(max_rows, rows * 4)
            t = self.step(rows)
        rows = max(16, min(max_rows, int(rows * target_s / max(t, 1e-3)) // 16 * 16))
        return rows

    def tops(self, rows: int, seconds: float) -> float:
        return 2.0 * rows * (D_FF * D_MODEL + D_MODEL * D_FF) / seconds / 1e12


def cpu_stages_child(rows: int) -> None:
    """Child process (CONVROT_THREADS fixed for its lifetime, parallel.cpp:10-22):
    the reference's stages on `rows` token rows of the fc1 / fc2 inputs --
    group_rotate, compute_scales + quantize, int_gemm -- and the whole
    forward_prepared, one warm-up and the median of 3 each."""
    import numpy as np
    ref = CpuReference(int(os.environ.get("CONVROT_THREADS", "1")))
    O = ref.O
    if ref.kind != "reference":
        print(json.dumps({"kind": ref.kind}))
        return
    x = ref.x_all[:rows]
    y1 = O.Ref.forward_prepared(x, ref.l1[0], ref.l1[1], ref.b1, O.ROT_REGULAR, N0)

    def med3(fn):
        fn()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts)

    out = {"kind": "reference", "threads": ref.threads, "rows": rows, "stages_s": {}}
    for name, xin, layer, k, n in (("fc1", x, ref.l1, D_MODEL, D_FF),
                                   ("fc2", y1, ref.l2, D_FF, D_MODEL)):
        rot = O.Ref.group_rotate(xin, O.ROT_REGULAR, N0)
        sc = O.Ref.compute_scales(rot, 4)
        codes = O.Ref.quantize(rot, sc, 4)
        out["stages_s"][name] = {
            "group_rotate": med3(lambda: O.Ref.group_rotate(xin, O.ROT_REGULAR, N0)),
            "compute_scales+quantize": med3(lambda: O.Ref.quantize(rot, O.Ref.compute_scales(rot, 4), 4)),
            "int_gemm": med3(lambda: O.Ref.int_gemm(codes, layer[0], 4, 4)),
            "forward": med3(lambda: O.Ref.forward_prepared(xin, layer[0], layer[1], None,
                                                           O.ROT_REGULAR, N0)),
        }
    fwd = out["stages_s"]["fc1"]["forward"] + out["stages_s"]["fc2"]["forward"]
    out["forward_s"] = fwd
    out["tops"] = 2.0 * rows * (D_FF * D_MODEL + D_MODEL * D_FF) / fwd / 1e12
    print(json.dumps(out), flush=True)


def cpu_baseline_staged(budget_s: float = 40.0):
    """The reference CPU path on the box's host cores, per BASELINE.md 3:
    CONVROT_THREADS = nproc and = 1 (each in its own process), per-stage
    times, one warm-up and the median of 3, on a bounded row sample (rows
    are independent: per-token scales).  ~budget_s of CPU work in total."""
    nproc = os.cpu_count() or 1
    res = {}
    # cost model: one forward of one row ~ 12 ms / nproc-thread-GOPS; each
    # child runs ~9 forward-equivalents (stages + forward, warm-up + 3)
    for threads, share in ((nproc, 0.6), (1, 0.4)):
        env = dict(os.environ, CONVROT_THREADS=str(threads))
        probe = subprocess.run([sys.executable, __file__, "--cpu-stages", "16"], env=env,
                               capture_output=True, text=True, timeout=600)
        try:
            p = json.loads(probe.stdout.strip().splitlines()[-1])
        except Exception:
            return {"value": None, "unit": "TOPS", "cores": 0, "kind": "unavailable",
                    "sample": f"cpu stage child failed: {probe.stderr[-300:]}"}
        if p.get("kind") != "reference":
            return None
        per_row = max(p["forward_s"] / 16, 1e-5)
        rows = int(max(16, min(1024, budget_s * share / 9.0 / per_row)) // 16 * 16)
        r = subprocess.run([sys.executable, __file__, "--cpu-stages", str(rows)], env=env,
                           capture_output=True, text=True, timeout=900)
        res[threads] = json.loads(r.stdout.strip().splitlines()[-1])
    top = res[nproc]
    one = res[1]
    return {"value": top["tops"], "unit": "TOPS", "cores": top["threads"], "kind": "reference",
            "sample": (f"{top['rows']} of {M_TOK} token rows through fc1+fc2 (forward_prepared), "
                       f"CONVROT_THREADS={top['threads']}; one warm-up, median of 3"),
            "stages_s": top["stages_s"],
            "threads_1": {"value": one["tops"], "unit": "TOPS", "rows": one["rows"],
                          "stages_s": one["stages_s"]}}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # N>1: rank 0 alone runs and prints
    threads = os.cpu_count() or 1
    ref = CpuReference(threads)
    rows = ref.calibrate(target_s=args.ref_seconds, max_rows=1024)
    for _ in range(args.warmup):
        ref.step(rows)
    times = [ref.step(rows) for _ in range(args.steps)]
    t = statistics.mean(times)
    v = ref.tops(rows, t)
    sample = (f"{rows} of {M_TOK} token rows through fc1+fc2 per step (rows are independent: "
              f"per-token scales); CONVROT_THREADS={ref.threads}")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TOPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int4", "data": "synthetic (seeded gaussian, bf16-representable)",
        "config": {"workload": WORKLOAD, "M": M_TOK, "d_model": D_MODEL, "d_ff": D_FF,
                   "n0": N0, "bits": "W4A4", "rows_per_step": rows},
        "cpu_baseline": {"value": v, "unit": "TOPS", "cores": ref.threads, "kind": ref.kind,
                         "sample": sample},
        "e2e": {"value": v, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        def reader():
            for line in self.proc.stdout:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == 7:
                    self.rows.append(parts)
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        def num(s):
            try:
                return float(s)
            except ValueError:
                return float("nan")
        sm = [num(r[0]) for r in self.rows]
        mx = [num(r[1]) for r in self.rows]
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower().startswith("active")})
        busy = [s for s in sm if not math.isnan(s)]
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# Per-config blocks (BASELINE.json configs[0], [2], [3]) and device-only
# kernel times: back-to-back launches captured in one CUDA graph, cycling
# over enough input buffers that every K1 launch reads its input from HBM
# (> 2x the 126 MB L2) -- launch gaps and host overhead excluded.
# ---------------------------------------------------------------------------
L2_BYTES = 126 * 1024 * 1024
NOMINAL_INT8_TOPS = 4500.0


def graph_us(calls, reps: int, dev) -> float:
    import torch
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        for c in calls:  # plans, attributes, tensor maps
            c()
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            for c in calls:
                c()
    g.replay()
    torch.cuda.synchronize(dev)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / (reps * len(calls)))
    del g
    return statistics.median(ts)


class KernelRig:
    """Device buffers for timing K1 (int8-code production layout) and K3 v3
    at one (M, K, N) through the C-ABI."""

    def __init__(self, lib, abi, dev, M, K, N=None, seed=5):
        import ctypes
        import torch
        self.lib, self.abi, self.dev, self.M, self.K, self.N = lib, abi, dev, M, K, N
        self.ct = ctypes
        g = torch.Generator(device=dev).manual_seed(seed)
        self.nbuf = max(2, -(-3 * L2_BYTES // (M * K * 2)))
        self.x = [torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
                  for _ in range(self.nbuf)]
        self.ld = (K + 15) // 16 * 16
        self.codes = [torch.empty(M, self.ld, dtype=torch.uint8, device=dev) for _ in range(self.nbuf)]
        self.s = [torch.empty(M, dtype=torch.float32, device=dev) for _ in range(self.nbuf)]
        self.sums = [torch.empty(M, dtype=torch.int32, device=dev) for _ in range(self.nbuf)]
        self.y = torch.empty(M, N or 1, dtype=torch.bfloat16, device=dev) if N else None

    def _sp(self):
        import torch
        return self.ct.c_void_p(torch.cuda.current_stream().cuda_stream)

    def k1(self, i, rc):
        P = lambda t: self.ct.c_void_p(t.data_ptr())  # noqa: E731
        self.abi.check(self.lib.crt_rotate_quant_i8(
            P(self.x[i]), self.abi.CRT_DTYPE_BF16, self.M, self.K, self.K, self.ct.byref(rc),
            P(self.codes[i]), self.ld, P(self.s[i]), P(self.sums[i]), self._sp()))

    def k3(self, i, layer):
        P = lambda t: self.ct.c_void_p(t.data_ptr())  # noqa: E731
        self.abi.check(self.lib.crt_quant_gemm_i8(
            P(self.codes[i]), self.ld, P(self.s[i]), P(self.sums[i]), layer.handle, self.M,
            self.abi.CRT_OUT_BF16, P(self.y), self.N, self._sp()))

    def k1_block(self, n0, hbm):
        from paper_2512_03673_b200 import RotationKind, RotationSpec
        rc = RotationSpec(RotationKind.regular, n0).c()
        us = graph_us([lambda i=i: self.k1(i, rc) for i in range(self.nbuf)],
                      max(2, 96 // self.nbuf), self.dev)
        packed = self.M * self.K * 2.5 + 4 * self.M  # SURVEY.md 8(d) algorithmic bytes
        moved = self.M * self.K * 3 + 8 * self.M      # int8 codes + scale + code sum
        return {"n0": n0, "us": us, "GBps_packed": packed / us / 1e3,
                "frac_packed": packed / us / 1e3 / hbm, "GBps_moved": moved / us / 1e3,
                "bytes_packed": packed}

    def k3_block(self, layer, int8_peak, n0):
        from paper_2512_03673_b200 import RotationKind, RotationSpec
        rc = RotationSpec(RotationKind.regular, n0).c()
        for i in range(self.nbuf):
            self.k1(i, rc)
        us = graph_us([lambda i=i: self.k3(i, layer) for i in range(self.nbuf)],
                      max(2, 24 // self.nbuf), self.dev)
        ops = 2 * self.M * self.N * self.K
        tops = ops / us / 1e6
        fwd = graph_us([c for i in range(self.nbuf)
                        for c in (lambda i=i: self.k1(i, rc), lambda i=i: self.k3(i, layer))],
                       max(2, 24 // self.nbuf), self.dev) * 2
        return {"k3_us": us, "k3_TOPS": tops, "k3_frac_measured_int8": tops / int8_peak,
                "k3_frac_nominal_int8": tops / NOMINAL_INT8_TOPS, "forward_us": fwd,
                "forward_TOPS": ops / fwd / 1e6}


def per_config_blocks(crt, lib, abi, dev, int8_peak, hbm):
    """cfg2's K1 roofline (both layers), cfg1 (attn-proj 4096x3072x3072),
    cfg3 (N0 sweep at 4608x3072x3072) and cfg4 (the FLUX.1-dev linear stack)."""
    import torch
    from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec
    out = {"timing": ("device-only: back-to-back launches in one CUDA graph over input buffers "
                      "> 2x L2 (every K1 reads HBM); forward = K1 + K3 pairs")}
    gw = torch.Generator(device=dev).manual_seed(7)
    # cfg2 K1 (the headline pair's rotate+quant kernels)
    out["cfg2_k1"] = {}
    for name, K in (("fc1", D_MODEL), ("fc2", D_FF)):
        rig = KernelRig(lib, abi, dev, M_TOK, K)
        out["cfg2_k1"][name] = rig.k1_block(N0, hbm)
        del rig
    # cfg1: single ConvLinear4bit forward, attn-proj M=4096, K=N=3072
    w = torch.randn(D_MODEL, D_MODEL, device=dev, generator=gw).to(torch.bfloat16)
    b = torch.randn(D_MODEL, device=dev, generator=gw)
    rig = KernelRig(lib, abi, dev, 4096, D_MODEL, D_MODEL)
    layer = crt.prepare_layer(w, b, RotationSpec(RotationKind.regular, N0), QuantSpec(4), "cfg1")
    out["cfg1"] = {"workload": "M=4096, K=N=3072, N0=16 (configs[0])", **rig.k1_block(N0, hbm),
                   **rig.k3_block(layer, int8_peak, N0)}
    del rig, layer
    # cfg3: N0 sweep at M=4608, K=N=3072
    rig = KernelRig(lib, abi, dev, M_TOK, D_MODEL, D_MODEL)
    sweep = []
    for n0 in (4, 16, 64, 256):
        layer = crt.prepare_layer(w, b, RotationSpec(RotationKind.regular, n0), QuantSpec(4), "cfg3")
        blk = rig.k1_block(n0, hbm)
        blk.update(rig.k3_block(layer, int8_peak, n0))
        sweep.append(blk)
        del layer
    out["cfg3"] = {"workload": "M=4608, K=N=3072, N0 in {4,16,64,256} (configs[2])",
                   "per_n0": sweep}
    del rig, w
    torch.cuda.empty_cache()
    # cfg4: the 494-linear FLUX.1-dev stack, siblings fused, text stream on a
    # second CUDA stream (paper_2512_03673_b200/flux.py)
    from paper_2512_03673_b200.flux import FluxStack, flux_linears, stack_ops
    ls = flux_linears()
    stk = FluxStack(ls, fused=True, n0=N0, streams=2, device=dev)
    for _ in range(2):
        stk.step()
    torch.cuda.synchronize(dev)
    graph = stk.capture()  # the step's 608 launches as one CUDA graph (no per-call host work)
    graph.replay()
    torch.cuda.synchronize(dev)
    ts = []
    for _ in range(5):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        e.record()
        e.synchronize()
        ts.append(a.elapsed_time(e))
    ms = statistics.median(ts)
    tops = stack_ops(ls) / (ms * 1e-3) / 1e12
    out["cfg4"] = {"workload": "FLUX.1-dev linear stack, 19 double + 38 single blocks, 494 linears "
                               "(304 fused units), N0=16, W4A4 (configs[3])",
                   "ms_per_step": ms, "TOPS": tops, "frac_measured_int8": tops / int8_peak,
                   "frac_nominal_int8": tops / NOMINAL_INT8_TOPS,
                   "device_layers_GiB": stk.layer_bytes / 2**30,
                   "timing": "median of 5 steps, CUDA events around each replay of the step's "
                             "CUDA graph (L2 warm)"}
    del graph, stk
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2512_03673_b200 as crt
    from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec, _abi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _abi.load()

    n0 = args.n0
    spec = RotationSpec(RotationKind.regular, n0)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    gw = torch.Generator(device=dev).manual_seed(99)  # same weights on every rank
    x = torch.randn(M_TOK, D_MODEL, device=dev, generator=g).to(torch.bfloat16)
    w1 = torch.randn(D_FF, D_MODEL, device=dev, generator=gw).to(torch.bfloat16)
    w2 = torch.randn(D_MODEL, D_FF, device=dev, generator=gw).to(torch.bfloat16)
    b1 = torch.randn(D_FF, device=dev, generator=gw)
    b2 = torch.randn(D_MODEL, device=dev, generator=gw)
    column = args.parallel in ("column", "colrow")  # world 1: a 1-rank communicator
    if column:
        # SURVEY.md 8e / configs[4] through the C-ABI tensor-parallel path
        from paper_2512_03673_b200.parallel import NcclComm, TensorParallelLinear
        comm = NcclComm()
        q4 = QuantSpec(4)
        tp1 = TensorParallelLinear(w1, b1, spec, q4, q4, "column", comm, "fc1")
        tp2 = TensorParallelLinear(w2, b2, spec, q4, q4,
                                   "row" if args.parallel == "colrow" else "column", comm, "fc2")
        fc1, fc2 = tp1.layer, tp2.layer
    else:
        fc1 = crt.prepare_layer(w1, b1, spec, QuantSpec(4), "fc1")
        fc2 = crt.prepare_layer(w2, b2, spec, QuantSpec(4), "fc2")
    del w1, w2
    n1, n2 = fc1.out_features, fc2.out_features  # per-rank columns (row: full N)

    # preallocated device buffers (no allocation in the timed region)
    # v3 (production forward): K1 writes one int8 per 4-bit code + per-row
    # code sums, K3 v3 expands the packed weights in hardware.  v2: K1 packs
    # two codes per byte, K3 v2 expands in software.
    v3 = args.path == "v3"
    cpb = 1.0 if v3 else 0.5  # activation code bytes per element
    ld1 = (int(D_MODEL * cpb) + 15) // 16 * 16
    ld2 = (int(D_FF * cpb) + 15) // 16 * 16
    c1 = torch.empty(M_TOK, ld1, dtype=torch.uint8, device=dev)
    c2 = torch.empty(M_TOK, ld2, dtype=torch.uint8, device=dev)
    s1 = torch.empty(M_TOK, dtype=torch.float32, device=dev)
    s2 = torch.empty(M_TOK, dtype=torch.float32, device=dev)
    r1 = torch.empty(M_TOK, dtype=torch.int32, device=dev)
    r2 = torch.empty(M_TOK, dtype=torch.int32, device=dev)
    rsum = {c1.data_ptr(): r1, c2.data_ptr(): r2}
    y1 = torch.empty(M_TOK, D_FF, dtype=torch.bfloat16, device=dev)
    y2 = torch.empty(M_TOK, D_MODEL, dtype=torch.bfloat16, device=dev)
    if column:
        ws_tp = crt.Workspace(M_TOK, D_FF, dev)
        y1s = torch.empty(M_TOK, n1, dtype=torch.bfloat16, device=dev)
        x2s = torch.empty(M_TOK, D_FF // world, dtype=torch.bfloat16, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    rc = spec.c()
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def k1(xin, codes, sc, K, ld):
        if v3:
            _abi.check(lib.crt_rotate_quant_i8(P(xin), _abi.CRT_DTYPE_BF16, M_TOK, K, K,
                                               ctypes.byref(rc), P(codes), ld, P(sc),
                                               P(rsum[codes.data_ptr()]), sp))
        else:
            _abi.check(lib.crt_rotate_quant(P(xin), _abi.CRT_DTYPE_BF16, M_TOK, K, K,
                                            ctypes.byref(rc), 4, P(codes), ld, P(sc), None, sp))

    def k3(codes, ld, sc, layer, y, N):
        if v3:
            _abi.check(lib.crt_quant_gemm_i8(P(codes), ld, P(sc), P(rsum[codes.data_ptr()]),
                                             layer.handle, M_TOK, _abi.CRT_OUT_BF16, P(y), N, sp))
        else:
            _abi.check(lib.crt_quant_gemm(P(codes), ld, P(sc), 4, layer.handle, M_TOK,
                                          _abi.CRT_OUT_BF16, P(y), N, sp))

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]

    def step(record):
        if column:  # C-ABI tensor-parallel forward of both layers
            if record:
                ev[0].record(stream)
            if args.parallel == "colrow":
                tp1(x, gather=False, y=y1s, workspace=ws_tp)   # [M, F/P]: fc2's input shard
                if record:
                    ev[2].record(stream)
                tp2(y1s, y=y2, workspace=ws_tp)                # int32 all-reduce -> [M, D]
            else:
                tp1(x, gather=True, y=y1, workspace=ws_tp)     # all-gather + interleave
                if record:
                    ev[2].record(stream)
                tp2(y1, gather=True, y=y2, workspace=ws_tp)
            if record:
                ev[4].record(stream)
            return
        if record:
            ev[0].record(stream)
        k1(x, c1, s1, D_MODEL, ld1)
        if record:
            ev[1].record(stream)
        k3(c1, ld1, s1, fc1, y1, D_FF)
        if record:
            ev[2].record(stream)
        k1(y1, c2, s2, D_FF, ld2)
        if record:
            ev[3].record(stream)
        k3(c2, ld2, s2, fc2, y2, D_MODEL)
        if record:
            ev[4].record(stream)

    for _ in range(max(3, args.warmup)):
        flush.zero_()
        step(False)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    launches0 = crt.launch_count()
    # Timed region: events only at the step boundaries, so consecutive
    # kernels overlap their launch / prologue with the predecessor's tail
    # (programmatic dependent launch, csrc/common.cuh).
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ms = []
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush, outside the event bracket
        es.record(stream)
        step(False)
        ee.record(stream)
        ee.synchronize()
        step_ms.append(es.elapsed_time(ee))
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    launches = crt.launch_count() - launches0
    # Per-kernel breakdown (kernels_us, roofline): the same K steps again with
    # an event between every kernel (which serialises them).
    seg = ({"fc1_tp": [], "fc2_tp": [], "step": []} if column else
           {"k1_fc1": [], "k3_fc1": [], "k1_fc2": [], "k3_fc2": [], "step": []})
    for _ in range(args.steps):
        flush.zero_()
        step(True)
        ev[4].synchronize()
        if column:
            seg["fc1_tp"].append(ev[0].elapsed_time(ev[2]))
            seg["fc2_tp"].append(ev[2].elapsed_time(ev[4]))
            seg["step"].append(ev[0].elapsed_time(ev[4]))
            continue
        seg["k1_fc1"].append(ev[0].elapsed_time(ev[1]))
        seg["k3_fc1"].append(ev[1].elapsed_time(ev[2]))
        seg["k1_fc2"].append(ev[2].elapsed_time(ev[3]))
        seg["k3_fc2"].append(ev[3].elapsed_time(ev[4]))
        seg["step"].append(ev[0].elapsed_time(ev[4]))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.stop()

    ms_step = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms_step], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    ops = layer_ops()
    # replicas: every rank runs the whole pair on its own prompt (weak);
    # column: the ranks share one pair (strong)
    value = (1 if column else world) * ops / (ms_step * 1e-3) / 1e12

    # roofline of the dominant kernel (K3), measured live on the launching stream
    if column:  # per-rank layer forward (K1 + K3 + collectives); no per-kernel split
        k3_us = (statistics.mean(seg["fc1_tp"]) + statistics.mean(seg["fc2_tp"])) / 2 * 1e3
    else:
        k3_us = (statistics.mean(seg["k3_fc1"]) + statistics.mean(seg["k3_fc2"])) / 2 * 1e3
    k3_ops_per_launch = 2 * M_TOK * D_FF * D_MODEL // (world if column else 1)
    k3_tops = k3_ops_per_launch / (k3_us * 1e-6) / 1e12
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    bf16_burst = float(peaks.get("bf16_tflops", 1590.0))
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    # the dense INT8 tensor ceiling measured directly (tools/probes/i8_peak_probe.cu,
    # profiles/int8_ceiling.json); 2 x the cuBLAS bf16 burst only if that file is absent
    int8_peak, int8_src = 2.0 * bf16_burst, "2 x measured bf16 burst (MEASURED_PEAKS.json)"
    try:
        int8_peak = float(json.load(open(os.path.join(ROOT, "profiles", "int8_ceiling.json")))[
            "kind_i8_tops"])
        int8_src = ("tcgen05 kind::i8 back-to-back MMA ceiling measured on this part "
                    "(tools/probes/i8_peak_probe.cu, profiles/int8_ceiling.json)")
    except Exception:
        pass
    # bf16 in + codes out + fp32 scale (+ int32 code sum for v3) per row
    k1_bytes = {k: M_TOK * kk * (2 + cpb) + (8 if v3 else 4) * M_TOK
                for k, kk in (("fc1", D_MODEL), ("fc2", D_FF))}
    k1_gbs = ({k: None for k in k1_bytes} if column else
              {k: k1_bytes[k] / (statistics.mean(seg[f"k1_{k}"]) * 1e-3) / 1e9 for k in k1_bytes})
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "k3_traffic.json"))).get(
            "fc1_bytes_per_launch")
    except Exception:
        pass

    # e2e through the public API with HOST buffers.  Every step copies its
    # input from pinned host memory, runs fc1 + fc2 and copies its result
    # back; steps are software-pipelined over NB streams / buffer sets (as a
    # serving loop would), so step k+1's upload and step k-1's download run
    # under step k's kernels.  Also reported: the unpipelined per-step latency.
    e2e = None
    if not args.no_e2e and not args.profile and not column:
        NB = 3
        xh = x.cpu().pin_memory()
        streams = [torch.cuda.Stream(dev) for _ in range(NB)]
        bufs = [{"xd": torch.empty_like(x),
                 "y1": torch.empty(M_TOK, D_FF, dtype=torch.bfloat16, device=dev),
                 "y2": torch.empty(M_TOK, D_MODEL, dtype=torch.bfloat16, device=dev),
                 "yh": torch.empty(M_TOK, D_MODEL, dtype=torch.bfloat16).pin_memory(),
                 "ws": crt.Workspace(M_TOK, D_FF, dev)} for _ in range(NB)]

        def e2e_step(k):
            b, st = bufs[k % NB], streams[k % NB]
            with torch.cuda.stream(st):
                b["xd"].copy_(xh, non_blocking=True)
                h = crt.forward(b["xd"], fc1, QuantSpec(4), out="bf16", y=b["y1"],
                                workspace=b["ws"], check_finite=False)
                o = crt.forward(h, fc2, QuantSpec(4), out="bf16", y=b["y2"], workspace=b["ws"],
                                check_finite=False)
                b["yh"].copy_(o, non_blocking=True)

        for k in range(2 * NB):
            e2e_step(k)
        torch.cuda.synchronize()
        n_e2e = max(3 * NB, args.steps)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        for st in streams[1:]:
            st.wait_event(e0)
        for k in range(n_e2e):
            e2e_step(k)
        ends = []
        for st in streams:
            ev_end = torch.cuda.Event(enable_timing=True)
            ev_end.record(st)
            ends.append(ev_end)
        torch.cuda.synchronize()
        e_ms = max(e0.elapsed_time(ev_end) for ev_end in ends) / n_e2e
        # unpipelined latency of one step (same copies, one stream)
        lat = []
        for k in range(NB):
            la, lb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            la.record(streams[0])
            e2e_step(0)
            lb.record(streams[0])
            lb.synchronize()
            lat.append(la.elapsed_time(lb))
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": world * ops / (e_ms * 1e-3) / 1e12, "unit": "TOPS",
               "h2d_bytes_per_step": xh.numel() * 2,
               "d2h_bytes_per_step": bufs[0]["yh"].numel() * 2,
               "ms_per_step": e_ms, "pipelined_streams": NB,
               "step_latency_ms": statistics.median(lat)}

    configs = None
    if rank == 0 and world == 1 and not args.no_configs and not args.profile:
        configs = per_config_blocks(crt, lib, _abi, dev, int8_peak, hbm)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        try:
            cpu = cpu_baseline_staged()
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "TOPS", "cores": 0, "kind": "unavailable",
                   "sample": f"error: {exc}"}

    if configs is not None:
        c2 = configs["cfg2_k1"]
        k1_roof = {"bound": "hbm", "kernel": "k1_team (rotate + quantise, int8 codes + row sums)",
                   "achieved": c2["fc2"]["GBps_packed"], "peak": hbm, "unit": "GB/s",
                   "frac": c2["fc2"]["frac_packed"], "fc1_gbs": c2["fc1"]["GBps_packed"],
                   "fc1_frac": c2["fc1"]["frac_packed"],
                   "bytes": "SURVEY.md 8(d): M*K*(2 B bf16 in + 0.5 B packed codes) + 4 B/row",
                   "us": {k: v["us"] for k, v in c2.items()},
                   "timing": configs["timing"]}
    else:
        k1_roof = {"bound": "hbm", "achieved": k1_gbs["fc2"], "peak": hbm, "unit": "GB/s",
                   "frac": k1_gbs["fc2"] / hbm if k1_gbs["fc2"] else None,
                   "fc1_gbs": k1_gbs["fc1"], "bytes_per_launch": k1_bytes,
                   "timing": ("not split out in tensor-parallel runs" if column else
                              "event-bracketed launches")}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if column else "weak",
            "vs_baseline": None, "dtype": "int4",
            "data": "synthetic (seeded gaussian bf16 activations, random-init weights)",
            "config": {"workload": WORKLOAD, "M": M_TOK, "d_model": D_MODEL, "d_ff": D_FF,
                       "n0": n0, "bits": "W4A4", "k3_path": ("int8 activation codes (K1 team -> K3 v4)" if v3 and
                                   os.environ.get("CRT_K3_V3") != "1" else args.path),
                       "parallelism": (
                           f"fc1 column-parallel (no gather) -> fc2 row-parallel (int32 SUM "
                           f"all-reduce) x{world}, C-ABI crt_tp_* over NCCL"
                           if column and args.parallel == "colrow" else
                           f"column-parallel x{world} + NCCL all-gather, C-ABI crt_tp_*"
                           if column else
                           f"prompt replicas x{world}" if world > 1 else "single"),
                       "l2": "flushed (256 MiB write) between steps, outside the timed events"},
            "roofline": {"bound": "tensor",
                         "kernel": ("per-rank tensor-parallel layer forward (K1 + K3 + NCCL); "
                                    "the ops are this rank's share" if column else
                                    "k3_v3_kernel (W4A4 GEMM, 2-SM tcgen05 kind::i8, weights "
                                    "expanded by tcgen05.cp decompression; CRT_K3_V3=1)"
                                    if os.environ.get("CRT_K3_V3") == "1" else
                                    "k3_v4_kernel (W4A4 GEMM, 2-SM tcgen05 kind::i8, packed "
                                    "weights TMA-staged, expanded into TMEM A by tcgen05.st)")
                                   if v3 else
                                   "k3_v2_kernel (W4A4 GEMM, 2-SM tcgen05 kind::i8, TMEM-A)",
                         "achieved": k3_tops, "peak": int8_peak, "unit": "TFLOP/s",
                         "frac": k3_tops / int8_peak, "traffic": traffic,
                         "traffic_source": ("dram__bytes_read.sum + dram__bytes_write.sum per fc1 "
                                            "launch from an ncu --set full capture "
                                            "(profiles/k3_traffic.json); not measured in this run"),
                         "peak_note": f"int8 dense = {int8_src}; "
                                      f"vs nominal 4500: {k3_tops / 4500:.3f}",
                         "ops_per_launch": k3_ops_per_launch, "avg_launch_us": k3_us},
            "k1_roofline": k1_roof,
            "kernels_us": {k: statistics.mean(v) * 1e3 for k, v in seg.items()},
            "kernels_note": "kernels_us and roofline.avg_launch_us come from a second pass of the "
                            "same steps with an event between kernels; ms_per_step from the timed "
                            "pass with events only at step boundaries (PDL overlap kept)",
            "configs": configs,
            "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
            "clocks": clocks.summary(), "wall_s_timed": wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.cpu_stages:
        cpu_stages_child(args.cpu_stages)
        return
    if args.impl == "reference":
        run_reference_arm(args)
        return
    run_ours(args)


if __name__ == "__main__":
    main()
