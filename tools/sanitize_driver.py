"""Small cases that reach every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck; one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_driver.py

Cases: the config-1 HOSVD (32^3: fill, INT8 shared-layout Gram, direct Jacobi, TTM, error), the
n = 2 and n = 4 grids, the row-scaled INT8 layout (k_i8_residues + k_i8_gemm on CTA pairs), the
DMMA Gram (k_gram_tma / k_gram_generic) and the DMMA fused Gram (k_gram_fused, cooperative grid),
the INT8 fused route, the cluster eigensolver (n = 512: k_rr_cluster, 4 CTAs), the SVD-accurate
HOSVD (k_cgs_block cooperative, k_block_dots, k_svd_cluster), Tucker-ALS, the symmetric path.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec  # noqa: E402


def main():
    T.load()
    only = sys.argv[1:]

    def want(name):
        return not only or name in only

    k = KernelSpec.matern(1.5, 0.3)
    if want("small"):
        for g, r in ((GridSpec.cube(32, 1.0), (8, 8, 8)), (GridSpec.cube(2, 1.0), (2, 2, 2)),
                     (GridSpec.cube(4, 1.0), (2, 2, 2)), (GridSpec((40, 36, 33), (-1.0,) * 3, (1.0,) * 3), (6, 5, 4))):
            F = T.fill(g, k)
            res = T.hosvd(g, r, F)
            T.error(g, r, F, res.U, res.core)
            T.hosvd(g, r, F, sync=False)
    g = GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    F = T.fill(g, KernelSpec.matern(0.7, 0.5))
    if want("rowscaled"):
        T.set_gram_engine(T.GRAM_INT8_ROWSCALED)
        T.hosvd(g, (12, 10, 9), F)
        T.set_gram_engine(T.GRAM_AUTO)
    if want("dmma"):
        T.set_gram_engine(T.GRAM_DMMA)
        T.hosvd(g, (12, 10, 9), F)
        g2 = GridSpec((40, 36, 33), (-1.0,) * 3, (1.0,) * 3)
        T.gram(g2, 2, T.fill(g2, k))
        gf = GridSpec.cube(128, 1.0)
        T.gram_fused(gf, k, 0)
        T.set_gram_engine(T.GRAM_AUTO)
    if want("fused"):
        gf = GridSpec.cube(128, 1.0)
        res = T.hosvd_fused(gf, k, (8, 8, 8))
        T.error_fused(gf, k, (8, 8, 8), res.U, res.core)
    if want("eig"):
        ge = GridSpec((512, 24, 24), (-1.0,) * 3, (1.0,) * 3)
        Fe = T.fill(ge, KernelSpec.matern(0.5, 0.1))
        G = T.gram(ge, 0, Fe)
        T.eig(G, 12)
    if want("accurate"):
        T.hosvd_accurate(g, (12, 10, 9), F)
    if want("als"):
        res = T.hosvd(g, (6, 5, 7), F)
        T.als(g, (6, 5, 7), F, res.U, 1)
    if want("sym"):
        T.hosvd_sym(GridSpec.cube(64, 1.0), k, (6, 6, 6))
    torch.cuda.synchronize()
    print("sanitize driver done")


if __name__ == "__main__":
    main()
