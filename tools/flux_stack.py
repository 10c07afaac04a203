"""Time the full FLUX.1-dev-shaped ConvLinear4bit stack (BASELINE.json
configs[3]: 19 double + 38 single blocks, 494 linears, 59.5 TOP/step,
random-init weights) on one GPU, unfused and with the f3 sibling fusion.
    python tools/flux_stack.py [--steps K] [--n0 16]
Prints one JSON line per variant."""
import argparse
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_03673_b200.flux import FluxStack, flux_linears, stack_ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--n0", type=int, default=16)
args = ap.parse_args()
ls = flux_linears()
ops = stack_ops(ls)
for fused, streams, graph in ((False, 1, False), (True, 1, False), (True, 2, False),
                              (True, 2, True)):
    st = FluxStack(ls, fused=fused, n0=args.n0, streams=streams)
    for _ in range(2):
        st.step()
    torch.cuda.synchronize()
    run = st.step
    if graph:
        g = st.capture()
        run = g.replay
        run()
        torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    print(json.dumps({"workload": "FLUX.1-dev linear stack 19 double + 38 single blocks (494 linears)",
                      "fused_siblings": fused, "cuda_streams": streams, "cuda_graph": graph,
                      "units": len(st.units), "n0": args.n0,
                      "ms_per_step": ms, "TOPS": ops / (ms * 1e-3) / 1e12,
                      "packed_weights_GiB": sum(l.n * ((l.k + 1) // 2) for l in ls) / 2**30,
                      "device_layers_GiB_measured": st.layer_bytes / 2**30}),
          flush=True)
    del st
    torch.cuda.empty_cache()
