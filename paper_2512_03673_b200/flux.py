"""FLUX.1-dev-shaped ConvLinear4bit stack (BASELINE.json configs[3]) and the
stack-level fusion of SURVEY.md 8f row f3.

The linear inventory of FLUX.1-dev at 1024x1024, batch 1 (image tokens
M = 4096, text tokens M = 512, single-stream M = 4608, AdaLN modulation on
the pooled embedding M = 1), d_model 3072, MLP 12288:

  19 double-stream blocks x 14 linears
     img: AdaLN 3072->18432 (M=1), q, k, v, out 3072->3072, fc1 3072->12288,
          fc2 12288->3072                                   (M = 4096)
     txt: the same seven                                    (M = 512)
  38 single-stream blocks x 6 linears
     AdaLN 3072->9216 (M=1), q, k, v 3072->3072, proj_mlp 3072->12288,
     proj_out 15360->3072                                   (M = 4608)
  = 494 linears, 59.5 TOP per step (2*M*N*K summed).

Fusion (f3): linears that read the same activations -- q/k/v of each stream,
and q/k/v/proj_mlp of a single block -- share one K1 (rotate + quantise the
input once) and run as ONE GEMM against the row-concatenated prepared
weights (N = 9216 or 21504).  Every output channel depends only on its own
weight row, scale and bias, and the activation codes / scales are the same,
so the fused outputs are bit-identical to the separate ones
(tests/test_flux_stack.py).

Streams: a double block's text-stream linears (M = 512) are independent of
its image-stream linears until the joint attention, and alone they fill
less than half of the GPU; with ``streams=2`` they run on a second CUDA
stream (own workspace) beside the image ones, joined at the end of the step.
Same kernels, same results.  Attention, norms and activations are not part of
the ConvLinear4bit path; the stack feeds each linear synthetic activations
of the right shape.
"""
from __future__ import annotations

import zlib
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import torch

from . import api

D, FF = 3072, 12288
M_IMG, M_TXT, M_SINGLE = 4096, 512, 4608


@dataclass(frozen=True)
class Linear:
    name: str
    m: int    # tokens
    k: int    # in_features
    n: int    # out_features
    group: str  # linears with the same group share their input (fusable)


def flux_linears(double_blocks: int = 19, single_blocks: int = 38, m_img: int = M_IMG,
                 m_txt: int = M_TXT, d: int = D, ff: int = FF) -> List[Linear]:
    out: List[Linear] = []
    for b in range(double_blocks):
        for s, m in (("img", m_img), ("txt", m_txt)):
            p = f"double{b}.{s}"
            out.append(Linear(f"{p}.adaln", 1, d, 6 * d, f"{p}.adaln"))
            for q in ("q", "k", "v"):
                out.append(Linear(f"{p}.{q}", m, d, d, f"{p}.qkv"))
            out.append(Linear(f"{p}.out", m, d, d, f"{p}.out"))
            out.append(Linear(f"{p}.fc1", m, d, ff, f"{p}.fc1"))
            out.append(Linear(f"{p}.fc2", m, ff, d, f"{p}.fc2"))
    m = m_img + m_txt
    for b in range(single_blocks):
        p = f"single{b}"
        out.append(Linear(f"{p}.adaln", 1, d, 3 * d, f"{p}.adaln"))
        for q in ("q", "k", "v"):
            out.append(Linear(f"{p}.{q}", m, d, d, f"{p}.in"))
        out.append(Linear(f"{p}.proj_mlp", m, d, ff, f"{p}.in"))
        out.append(Linear(f"{p}.proj_out", m, d + ff, d, f"{p}.proj_out"))
    return out


def stack_ops(linears: List[Linear]) -> int:
    return sum(2 * l.m * l.n * l.k for l in linears)


class FluxStack:
    """All linears prepared on one GPU (random-init bf16 weights, seeded),
    either one layer per linear or fused per input group."""

    def __init__(self, linears: List[Linear], fused: bool, n0: int = 16, bits: int = 4,
                 device="cuda", seed: int = 2, streams: int = 1):
        self.linears, self.fused, self.device = linears, fused, torch.device(device)
        self.streams = streams
        self.spec = api.RotationSpec(api.RotationKind.regular, n0)
        self.q = api.QuantSpec(bits)
        groups: Dict[str, List[Linear]] = {}
        for l in linears:
            groups.setdefault(l.group if fused else l.name, []).append(l)
        self.units: List[Tuple[List[Linear], api.PreparedLayer]] = []
        g = torch.Generator(device=self.device)
        # device memory the prepared layers own (cudaMalloc'd by the library,
        # outside torch's caching allocator): free-memory drop minus torch's
        # own reserve growth (the random bf16 weights are torch tensors)
        torch.cuda.synchronize(self.device)
        free0, res0 = torch.cuda.mem_get_info(self.device)[0], torch.cuda.memory_reserved(self.device)
        for i, (key, ls) in enumerate(groups.items()):
            ws, bs = [], []
            for l in ls:
                g.manual_seed(seed + zlib.crc32(l.name.encode()))
                ws.append(torch.randn(l.n, l.k, device=self.device, generator=g)
                          .mul_(l.k ** -0.5).to(torch.bfloat16))
                bs.append(torch.randn(l.n, device=self.device, generator=g).mul_(0.01))
            w = torch.cat(ws, 0) if len(ws) > 1 else ws[0]
            b = torch.cat(bs, 0) if len(bs) > 1 else bs[0]
            self.units.append((ls, api.prepare_layer(w, b, self.spec, self.q, key)))
            del w, ws
        torch.cuda.synchronize(self.device)
        self.layer_bytes = ((free0 - torch.cuda.mem_get_info(self.device)[0])
                            - (torch.cuda.memory_reserved(self.device) - res0))
        # one synthetic input per (M, K) shape, reused by every linear of that shape
        self.inputs: Dict[Tuple[int, int], torch.Tensor] = {}
        for ls, _ in self.units:
            key = (ls[0].m, ls[0].k)
            if key not in self.inputs:
                g.manual_seed(seed + 7 * key[0] + key[1])
                self.inputs[key] = torch.randn(*key, device=self.device, generator=g).to(
                    torch.bfloat16)
        self.ws = api.Workspace(max(l.m for l in linears), max(l.k for l in linears),
                                self.device)
        if streams > 1:
            self.side = torch.cuda.Stream(self.device)
            self.ws_side = api.Workspace(max(l.m for l in linears), max(l.k for l in linears),
                                         self.device)
        self.outputs = {id(u): torch.empty(u[0][0].m, u[1].out_features, dtype=torch.bfloat16,
                                           device=self.device) for u in self.units}

    def step(self) -> None:
        if self.streams == 1:
            for u in self.units:
                ls, layer = u
                x = self.inputs[(ls[0].m, ls[0].k)]
                api.forward(x, layer, self.q, out="bf16", y=self.outputs[id(u)],
                            workspace=self.ws, check_finite=False)
            return
        main = torch.cuda.current_stream(self.device)
        self.side.wait_stream(main)
        for u in self.units:
            ls, layer = u
            x = self.inputs[(ls[0].m, ls[0].k)]
            txt = ".txt." in ls[0].name
            with torch.cuda.stream(self.side if txt else main):
                api.forward(x, layer, self.q, out="bf16", y=self.outputs[id(u)],
                            workspace=self.ws_side if txt else self.ws, check_finite=False)
        main.wait_stream(self.side)

    def capture(self) -> "torch.cuda.CUDAGraph":
        """One CUDA graph of step() (both streams): every forward's K1 / K3
        launches replayed without the per-call host work (the stack's 304
        Python calls otherwise leave the GPU waiting on small units)."""
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.step()  # warm (tensor maps, smem attributes) outside the capture
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.step()
        return g

    def output_of(self, name: str) -> Optional[torch.Tensor]:
        """The output columns of linear `name` (a view into its unit's output)."""
        for u in self.units:
            ls, _ = u
            off = 0
            for l in ls:
                if l.name == name:
                    return self.outputs[id(u)][:, off:off + l.n]
                off += l.n
        return None
