"""A/B timing of K1 (int8-code mode, N0=16, bf16) between package copies.
    python tools/k1_ab.py ROOT_A ROOT_B [rounds]
Each ROOT holds a built paper_2512_03673_b200/ package; every (root, shape)
is timed in its own subprocess, rounds interleaved A/B/A/B, and the outputs
of the two roots are compared for equality."""
import subprocess
import sys

CHILD = r'''
import sys, hashlib, torch
sys.path.insert(0, sys.argv[1])
import paper_2512_03673_b200 as crt
from paper_2512_03673_b200 import RotationKind, RotationSpec
M, K = int(sys.argv[2]), int(sys.argv[3])
torch.manual_seed(0)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
spec = RotationSpec(RotationKind.regular, 16)
c8, s8, sums = crt.rotate_quantize_i8(x, spec)
h = hashlib.md5(c8.cpu().numpy().tobytes() + s8.cpu().numpy().tobytes() + sums.cpu().numpy().tobytes()).hexdigest()[:12]
flush = torch.empty(64 * 1024 * 1024, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for i in range(105):
    flush.zero_()
    ev[0].record()
    crt.rotate_quantize_i8(x, spec)
    ev[1].record()
    ev[1].synchronize()
    if i >= 5:
        ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
# single-launch event times are quantised; the mean of 100 varies in phase
print(f"{sum(ts) / len(ts):.2f} {h}")
'''


def main():
    roots = sys.argv[1:3]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    for M, K in [(4608, 3072), (4608, 12288)]:
        res = {r: [] for r in roots}
        hashes = {}
        for _ in range(rounds):
            for r in roots:
                out = subprocess.run([sys.executable, "-c", CHILD, r, str(M), str(K)],
                                     capture_output=True, text=True)
                if out.returncode:
                    print(out.stderr[-2000:])
                    raise SystemExit(1)
                t, h = out.stdout.split()
                res[r].append(float(t))
                hashes[r] = h
        same = len(set(hashes.values())) == 1
        print(f"M={M} K={K} same_output={same} " +
              "  ".join(f"{r}: {min(v):.2f} us (runs {v})" for r, v in res.items()), flush=True)


if __name__ == "__main__":
    main()
