"""A prepared layer is immutable and shareable (SPEC.md:289 in the reference;
include/crt/convlinear4bit.h): forwards from several host threads, each on
its own CUDA stream and workspace, give the single-threaded results.  The
ctypes calls release the GIL, so the launchers really run concurrently."""
import threading

import pytest
import torch


@pytest.mark.gpu
def test_forward_from_threads_on_own_streams():
    import paper_2512_03673_b200 as crt
    from paper_2512_03673_b200 import QuantSpec, RotationKind, RotationSpec
    g = torch.Generator(device="cuda").manual_seed(5)
    spec = RotationSpec(RotationKind.regular, 16)
    w = torch.randn(768, 3072, device="cuda", generator=g).to(torch.bfloat16)
    layer = crt.prepare_layer(w, torch.randn(768, device="cuda", generator=g), spec)
    layer8 = crt.prepare_layer(w, None, spec, QuantSpec(8))
    xs = [torch.randn(m, 3072, device="cuda", generator=g).to(torch.bfloat16)
          for m in (1, 200, 4096)]
    want = [(crt.forward(x, layer), crt.forward(x, layer8, QuantSpec(8))) for x in xs]
    torch.cuda.synchronize()
    errors = []

    def worker(tid):
        try:
            st = torch.cuda.Stream()
            ws = crt.Workspace(4096, 3072)
            with torch.cuda.stream(st):
                for it in range(8):
                    i = (tid + it) % len(xs)
                    y4 = crt.forward(xs[i], layer, workspace=ws)
                    y8 = crt.forward(xs[i], layer8, QuantSpec(8), workspace=ws)
                    st.synchronize()
                    if not (torch.equal(y4, want[i][0]) and torch.equal(y8, want[i][1])):
                        errors.append((tid, it))
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
