"""Is the C4 Llama step run-to-run deterministic (the precondition of the
byte-identity check against the no-offload step)?  Runs two fresh 4-step
sequences and compares losses + state checksums; reports the attention
kernels used.  python tools/det_probe.py [8b|tiny] [det]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
if "det" in sys.argv:
    os.environ["CUBLAS_WORKSPACE_CONFIG"] = ":4096:8"
import torch  # noqa: E402

from paper_2506_06472_b200 import engine  # noqa: E402
from paper_2506_06472_b200.llama_step import LLAMA3_8B_MODEL, TINY, Step  # noqa: E402

if "det" in sys.argv:
    torch.use_deterministic_algorithms(True, warn_only=True)
cfg = LLAMA3_8B_MODEL if "8b" in sys.argv else TINY


import contextlib  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

BACKEND = {"flash": SDPBackend.FLASH_ATTENTION, "efficient": SDPBackend.EFFICIENT_ATTENTION,
           "math": SDPBackend.MATH}
def ctx():
    b = next((BACKEND[a] for a in sys.argv if a in BACKEND), None)
    return sdpa_kernel(b) if b is not None else contextlib.nullcontext()


if "cudnndet" in sys.argv:
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False


def seq():
    s = Step(cfg, seed=0)
    import time
    with ctx():
        s()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        losses = [s().item() for _ in range(3)]
        print("ms/step", (time.perf_counter() - t0) / 3 * 1e3)
    g = s.globals_of()
    cs = engine.checksums([g[n] for n in sorted(g)])
    del s, g
    torch.cuda.empty_cache()
    return losses, cs


a = seq()
b = seq()
print("losses", a[0], b[0], "equal", a[0] == b[0], "checksums equal", a[1] == b[1],
      "n_diff", sum(x != y for x, y in zip(a[1], b[1])), "of", len(a[1]))
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as p:
    s = Step(cfg, seed=0)
    with ctx():
        s()
    torch.cuda.synchronize()
names = sorted({e.name for e in p.events() if "attn" in e.name.lower() or "fmha" in e.name.lower()
                or "flash" in e.name.lower() or "sdpa" in e.name.lower() or "cudnn" in e.name.lower()})
print("attention kernels:", names[:12])
