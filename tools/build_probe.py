"""Build tools/gemm_probe{1,3} (diagnostics only): the library's GEMM translation unit compiled with each
mbarrier wait strategy (LG_MBAR_MODE 1 = try_wait (default), 3 = bounded wait reporting stuck barriers)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2109_11978_b200 import build as B  # noqa: E402

inc, _ = B._nccl_dirs()
rc = 0
for mode in (1, 3):
    obj = os.path.join(B.BUILD, f"gemm_tc_probe{mode}.o")
    cmd = [B.NVCC, *B.FLAGS, f"-DLG_MBAR_MODE={mode}", "-I", os.path.join(ROOT, "include"), "-c",
           os.path.join(B.CSRC, "gemm_tc.cu"), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[-3000:])
        sys.exit(1)
    cmd = [B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tools", "gemm_probe.cu"), obj, "-lcuda", "-o", os.path.join(ROOT, "tools", f"gemm_probe{mode}")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[-3000:])
        rc = 1
sys.exit(rc)
