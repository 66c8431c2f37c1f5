"""Tile-shape comparison at every cascade width (M = width x 4680 rows):
single-CTA 128x128 / 128x256 tiles vs CTA-pair 256x192 / 256x256 tiles,
for the N = 1536 / 4608 / 8960 projections (calibrates gemm_plan)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gemm_bench.py")).read().split("for (M,Nn,K)")[0])
for w in (1, 2, 3, 4, 5):
    M = 4680 * w
    for (Nn, K, mode) in ((1536, 1536, 3), (4608, 1536, 0), (8960, 1536, 1), (1536, 8960, 3)):
        for bn, cg in ((128, 1), (256, 1), (192, 2), (256, 2), (0, 0)):
            if Nn % (bn or 64):
                continue
            run(M, Nn, K, mode, bn, cg=cg, iters=10)
