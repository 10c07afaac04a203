"""Per-shape time breakdown of the fused FLUX stack (dev aid): each unit's
forward timed alone (events around it), summed by (M, K, N)."""
import collections
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_03673_b200 import api  # noqa: E402
from paper_2512_03673_b200.flux import FluxStack, flux_linears  # noqa: E402

st = FluxStack(flux_linears(), fused=True)
st.step()
torch.cuda.synchronize()
acc = collections.defaultdict(lambda: [0, 0.0, 0])
for rep in range(2):
    for u in st.units:
        ls, layer = u
        x = st.inputs[(ls[0].m, ls[0].k)]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        api.forward(x, layer, st.q, out="bf16", y=st.outputs[id(u)], workspace=st.ws, check_finite=False)
        b.record()
        b.synchronize()
        if rep == 1:
            key = (ls[0].m, ls[0].k, layer.out_features)
            acc[key][0] += 1
            acc[key][1] += a.elapsed_time(b)
            acc[key][2] += 2 * ls[0].m * ls[0].k * layer.out_features
tot = sum(v[1] for v in acc.values())
print(f"total {tot:.2f} ms")
for k, (n, ms, ops) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"M={k[0]:5d} K={k[1]:5d} N={k[2]:5d} x{n:3d}: {ms:7.2f} ms ({ms / tot * 100:4.1f}%) "
          f"{ops / (ms * 1e-3) / 1e12:7.0f} TOPS  {ms / n * 1e3:7.1f} us/unit")
