"""int8 tcgen05 GEMM microbenchmark through tango_gemm_q (bench.py's `tensor` field):
python tools/gemm_bench.py [size] — prints achieved int8 TOPS vs the int8 tensor peak."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2308_00890_b200 import tango as T  # noqa: E402

if __name__ == "__main__":
    T.load()
    peaks, _ = bench.load_peaks()
    size = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    print(bench.gemm_microbench(T, torch, 2.0 * peaks["bf16_tflops"], size=size, reps=5))
