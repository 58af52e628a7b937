"""Time the lifetime stage alone (CUDA events, L2 flushed before each call)
for one or more builds of libtio: python tools/time_lifetime.py c3 lib1.so ..."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2506_06472_b200 import _native
    import bench
    cfg = sys.argv[1]
    tr, cap, rates, hc, desc = bench._trace(cfg)
    a = tr.arrays()
    for so in sys.argv[2:]:
        _native._lib = None
        _native.lib_path = lambda so=so: so
        lib = _native.load(build_if_missing=False)
        s = torch.cuda.Stream()
        dt = _native.DeviceTrace(a, stream=s.cuda_stream)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        ts = []
        for i in range(8):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            _native.check(lib.tio_lifetime(dt.handle, ctypes.c_void_p(s.cuda_stream)))
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts = sorted(ts[2:])
        import hashlib
        import numpy as np
        out = dt.lifetime()
        h = hashlib.sha256(b"".join(np.ascontiguousarray(np.asarray(out[k])).tobytes() for k in
                                    ("timeline", "active", "period_tensor", "period_start", "period_end",
                                     "period_wraps"))).hexdigest()[:16]
        print(os.path.basename(so), cfg, "lifetime ms min %.4f med %.4f" % (ts[0], ts[len(ts) // 2]), h,
              flush=True)


if __name__ == "__main__":
    main()
