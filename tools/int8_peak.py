"""Measured int8 tensor-core peak on this B200 (the fused filter's roofline
denominator): torch._int_mm (cuBLASLt IMMA) on square int8 GEMMs, CUDA
events, best of 10 after warm-up; writes profiles/int8_peak.json."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    torch.cuda.init()
    res = {}
    for n in (4096, 8192, 16384):
        a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()  # column-major B
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res[str(n)] = 2.0 * n ** 3 / (best / 1e3) / 1e12
        print(f"int8 {n}^3: {best:.3f} ms = {res[str(n)]:.1f} TOP/s", flush=True)
    out = {"int8_tops": max(res.values()), "per_size_tops": res,
           "how": "torch._int_mm (cuBLASLt int8 IMMA, s32 out), square n^3, 2*n^3 ops, best of 10 "
                  "CUDA-event timings after 3 warm-ups", "gpu": torch.cuda.get_device_name()}
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "int8_peak.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
