"""Measure the FP64 roofline denominators on a B200 (MEASURED_PEAKS.json has none):
  * cuBLAS DGEMM via torch.matmul float64 8192^3 (best of 10, and 4 s back to back),
  * FFMA.F64 and DMMA (mma.sync m8n8k4 f64) chains from tools/fp64_peak.cu,
and write profiles/fp64_peaks.json.  Run on the GPU box:  python tools/fp64_peak.py
"""
import json
import os
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    out = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) * 1e-3))
    out["dgemm_tflops"] = best / 1e12
    t0 = time.time()
    cnt = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b)
        cnt += 1
        if cnt % 8 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    out["dgemm_tflops_sustained"] = cnt * 2 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    if not os.path.exists(exe):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-o", exe, os.path.join(ROOT, "tools", "fp64_peak.cu")])
    micro = json.loads(subprocess.check_output([exe]).decode())
    out.update(micro)
    out["how"] = ("torch.matmul float64 8192^3 (cuBLAS DGEMM) best of 10 and 4 s back to back; "
                  "tools/fp64_peak.cu FFMA.F64 chains (8 accumulators/thread, 148x8 CTAs x 256) and "
                  "mma.sync m8n8k4 f64 chains (4 accumulators/warp), best of 4 after warm-up")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "profiles", "fp64_peaks.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
