import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_1711_06874_b200 import tucker as T
from tucker_inputs import GridSpec, KernelSpec
for g, k, chunk in [(GridSpec.cube(128), KernelSpec.matern(1.5, 0.2), None),
                    (GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)), KernelSpec.matern(0.7, 0.5), "256"),
                    (GridSpec((144, 136, 130), (-0.5, -2.0, 0.1), (1.5, 1.0, 0.9)), KernelSpec.matern(1.5, 0.2), "300"),
                    (GridSpec.cube(256), KernelSpec.matern(1.5, 0.2), "1024"),
                    (GridSpec.cube(1024), KernelSpec.matern(1.5, 0.2), None)]:
    if chunk: os.environ["TUCKER_FUSED_CHUNK_KB"] = chunk
    else: os.environ.pop("TUCKER_FUSED_CHUNK_KB", None)
    F = T.fill(g, k)
    ws = T.workspace(g)
    wsf = T.workspace_fused(g)
    for m in range(3):
        G = T.gram(g, m, F, ws)
        torch.cuda.synchronize(); t0 = time.time()
        Gf = T.gram_fused(g, k, m, wsf)
        torch.cuda.synchronize(); t1 = time.time()
        d = torch.sqrt(torch.diag(G))
        rel = ((Gf - G).abs() / torch.outer(d, d)).max().item()
        print(g.n, m, f"rel {rel:.2e} sym {torch.equal(Gf, Gf.T)} {1e3*(t1-t0):.2f} ms", flush=True)
    del F, ws, wsf
    torch.cuda.empty_cache()
