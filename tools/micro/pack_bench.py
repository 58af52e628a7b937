"""k_pack (the engine's TMA gather into 4 KB-aligned staging extents,
csrc/engine.cu) against the HBM roofline: 2 x bytes (read + write) over the
CUDA-event time (device work only: a spin kernel ahead of the timed region
covers the host's enqueue), best of 10, vs MEASURED_PEAKS.json hbm_gbs;
beside it one cudaMemcpyAsync D2D per tensor (the alternative).  One JSON
line per case."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2506_06472_b200 import engine
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    s = torch.cuda.current_stream()
    for n, size in ((256, 4 << 20), (4096, 256 << 10), (16384, 16 << 10)):
        ts = [torch.randint(0, 255, (size,), dtype=torch.uint8, device="cuda") for _ in range(n)]
        total = n * size
        staging = torch.empty(sum((size + 4095) // 4096 * 4096 for _ in range(n)), dtype=torch.uint8, device="cuda")
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            # a ~2 ms spin first, so the host finishes enqueueing the pack
            # before the GPU reaches it: the events then time the device work
            torch.cuda._sleep(4_000_000)
            e0.record(s)
            offs = engine.pack(ts, staging, stream=s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        ok = all(torch.equal(staging[o:o + size], t) for o, t in zip(offs[:64], ts[:64]))
        best_cp = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            torch.cuda._sleep(40_000_000)
            e0.record(s)
            for o, t in zip(offs, ts):
                staging[o:o + size].copy_(t)
            e1.record(s)
            torch.cuda.synchronize()
            best_cp = min(best_cp, e0.elapsed_time(e1))
        gbs = 2 * total / (best * 1e6)
        print(json.dumps({"tensors": n, "bytes_each": size, "total_bytes": total, "pack_ms": best,
                          "pack_gbs_rw": gbs, "frac_of_hbm_peak": gbs / peak, "hbm_peak_gbs": peak,
                          "per_tensor_copy_ms": best_cp, "per_tensor_copy_gbs_rw": 2 * total / (best_cp * 1e6),
                          "bytes_ok": ok}), flush=True)
        del ts, staging
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
