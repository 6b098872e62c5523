"""tucker_eig on a 1024 x 1024 Matérn Gram (mode 0 of a 1024 x 64 x 64 grid), for ncu captures of
the eigensolver kernels; prints the solve's time and info."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    r = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    T.load()
    g = GridSpec((n, 64, 64), (-1.0,) * 3, (1.0,) * 3)
    F = T.fill(g, KernelSpec.matern(1.5, 0.2))
    G = T.gram(g, 0, F)
    for _ in range(2):
        U, lam, info, rc = T.eig(G, r)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        U, lam, info, rc = T.eig(G, r)
    b.record()
    torch.cuda.synchronize()
    print("eig ms", a.elapsed_time(b) / 5, "rc", rc, info)


if __name__ == "__main__":
    main()
