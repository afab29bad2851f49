"""L2-chunking probe: would running each 24,576-row minibatch as L2-sized row chunks pay?

An iteration with K_mb = 4, 8, 12, 16 minibatches runs the same update GEMM chain on 24,576, 12,288, 8,192, 6,144
rows per launch: at K_mb = 12 every launch sees exactly the 8,192-row chunk the chunked plan would run (its ~56 MB
of activations stay in the 126 MB L2), so the per-category serialised GEMM times (profiled graph replay) are the
chunked plan's cost without its savings on Adam (one Adam per minibatch either way). C3 world, 4096 x 24.

usage: python tools/chunk_probe.py > gpurun_out/chunk_probe.txt"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import bench  # noqa: E402
import sweep  # noqa: E402
from paper_2109_11978_b200 import lg  # noqa: E402


def main():
    torch.cuda.set_device(0)
    hfd = torch.empty((800, 1600), device="cuda")
    lg.lg_terrain_generate(hfd, 10, 20, 11)
    torch.cuda.synchronize()
    hf = hfd.cpu().numpy()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for k in (4, 8, 12, 16):
        r = sweep.point(hf, 4096, 24, k, 10, flush, bench.peaks())
        print(k, round(r["ms_median"], 3), r["phase_ms"], flush=True)


if __name__ == "__main__":
    main()
