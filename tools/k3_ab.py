"""A/B timing of K3 v3 (W4A4, bf16 out) at the FLUX shapes between built
package copies: python tools/k3_ab.py ROOT_A ROOT_B [rounds].  Each
(root, round) runs in its own process; outputs are compared by digest."""
import subprocess
import sys

CHILD = r'''
import sys, hashlib, torch
sys.path.insert(0, sys.argv[1])
import paper_2512_03673_b200 as crt
from paper_2512_03673_b200 import RotationKind, RotationSpec
spec = RotationSpec(RotationKind.regular, 16)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
out = []
for M, K, N in [(4608, 3072, 12288), (4608, 12288, 3072)]:
    torch.manual_seed(0)
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    layer = crt.prepare_layer(torch.randn(N, K, device="cuda").to(torch.bfloat16), None, spec)
    c, sa, su = crt.rotate_quantize_i8(x, spec)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(43):
        flush.zero_()
        s.record()
        crt.quant_gemm_i8(c, sa, su, layer, y=y)
        e.record()
        e.synchronize()
        if i >= 3:
            ts.append(s.elapsed_time(e) * 1e3)
    h = hashlib.md5(y.view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:10]
    out.append(f"{sum(ts) / len(ts):.1f}:{h}")
print(" ".join(out))
'''


def main():
    roots = sys.argv[1:3]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    for _ in range(rounds):
        for r in roots:
            p = subprocess.run([sys.executable, "-c", CHILD, r], capture_output=True, text=True)
            print(r, p.stdout.strip() if p.returncode == 0 else p.stderr[-1500:], flush=True)


if __name__ == "__main__":
    main()
