"""Floor of the lifetime stage's scattered RED atomics on the C3 trace.

    python tools/micro/red_floor.py [c3|c2]

Builds tools/micro/libred_floor.so, uploads the trace's access column, CSR
offsets and kinds, and times (CUDA events, best of 10, L2 flushed) the
red_floor.cu modes: access-column stream only; one RED.64 per event
(per_kernel_active_bytes); plus the difference-array REDs (k_events' full
atomic traffic); 32-bit REDs.  Prints one JSON line.
"""

import ctypes
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2506_06472_b200 import tracegen as G
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    so = os.path.join(HERE, "libred_floor.so")
    if not os.path.exists(so):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                        "-fPIC", os.path.join(HERE, "red_floor.cu"), "-o", so], check=True)
    L = ctypes.CDLL(so)
    tr = G.gen_llama_trace(G.LLAMA3_70B if cfg == "c3" else G.LLAMA3_8B)
    a = tr.arrays()
    dev = torch.device("cuda")
    acc = torch.from_numpy(a.accesses.astype("int32")).to(dev)
    ptr = torch.from_numpy(a.access_ptr.astype("int64")).to(dev)
    kind = torch.from_numpy(a.kind.astype("int8")).to(dev)
    N, T, E = a.num_kernels, a.num_tensors, a.num_events
    act = torch.zeros(N + 2, dtype=torch.int64, device=dev)
    dif = torch.zeros(N + 2, dtype=torch.int64, device=dev)
    inter = int((a.kind == 0).sum())
    out = {"config": cfg, "events": E, "kernels": N, "tensors": T, "intermediates": inter}
    names = {0: "stream_acc_only", 1: "red64_per_event", 2: "red64_per_event_plus_diff", 3: "red32_per_event"}
    for mode in (0, 1, 2, 3):
        ms = ctypes.c_float()
        rc = L.red_floor(ctypes.c_void_p(acc.data_ptr()), ctypes.c_void_p(ptr.data_ptr()),
                         ctypes.c_void_p(kind.data_ptr()), ctypes.c_int64(E), ctypes.c_int64(T), ctypes.c_int64(N),
                         ctypes.c_void_p(act.data_ptr()), ctypes.c_void_p(dif.data_ptr()), mode, 10,
                         ctypes.byref(ms))
        assert rc == 0, rc
        out[names[mode] + "_us"] = ms.value * 1e3
    out["reds_per_event_pass"] = E
    out["reds_diff"] = 2 * inter
    print(json.dumps(out))


if __name__ == "__main__":
    main()
