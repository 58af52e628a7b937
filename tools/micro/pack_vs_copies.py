"""When does the engine's TMA pack kernel pay on the offload path?  n tensors
of `size` bytes moved to pinned host memory (a) one cudaMemcpyAsync D2H per
tensor, (b) k_pack into one 4 KB-aligned device staging extent + one D2H of
the extent.  CUDA-event times (device work only: a spin kernel ahead covers
the host's enqueue), best of 5.  One JSON line per size."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2506_06472_b200 import engine
    s = torch.cuda.current_stream()
    total = 256 << 20
    for size in (4 << 10, 16 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20):
        n = total // size
        ts = [torch.randint(0, 255, (size,), dtype=torch.uint8, device="cuda") for _ in range(n)]
        ext = (size + 4095) // 4096 * 4096
        staging = torch.empty(n * ext, dtype=torch.uint8, device="cuda")
        host = torch.empty(n * ext, dtype=torch.uint8, pin_memory=True)

        def timed(fn, reps=5):
            best = 1e9
            for _ in range(reps):
                torch.cuda.synchronize()
                torch.cuda._sleep(20_000_000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                fn()
                e1.record(s)
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            return best

        def copies():
            for i, t in enumerate(ts):
                host[i * ext:i * ext + size].copy_(t, non_blocking=True)

        def packed():
            engine.pack(ts, staging, stream=s.cuda_stream)
            host.copy_(staging, non_blocking=True)

        a, b = timed(copies), timed(packed)
        print(json.dumps({"tensor_bytes": size, "tensors": n, "total_bytes": n * size,
                          "per_tensor_copies_ms": a, "pack_plus_one_copy_ms": b,
                          "per_tensor_gbs": n * size / (a * 1e6), "packed_gbs": n * size / (b * 1e6)}), flush=True)
        del ts, staging, host
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
