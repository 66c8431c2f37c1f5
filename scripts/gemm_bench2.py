"""Tile-width comparison on the Wan-1.3B width-5 shapes (M = 23,400):
256- vs 192-column CTA-pair tiles and the automatic choice, plus the GELU
epilogue."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gemm_bench.py")).read().split("for (M,Nn,K)")[0])
for (M, Nn, K, mode) in [(23400, 1536, 1536, 3), (23400, 1536, 8960, 3), (23400, 1536, 1536, 0),
                         (23400, 4608, 1536, 0), (23400, 8960, 1536, 1), (23400, 8960, 1536, 0),
                         (4680, 1536, 1536, 3), (18720, 1536, 8960, 3)]:
    for bn, cg in ((256, 2), (192, 2), (0, 0)):
        if Nn % (bn or 64):
            continue
        run(M, Nn, K, mode, bn, cg=cg)
