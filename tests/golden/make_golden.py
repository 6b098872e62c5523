"""Writes the oracle golden files for the full-size parity tests (tests/test_gpu_target.py).

Calls ONLY ``oracle/`` (plain C, Dot2 Gram, cyclic Jacobi — test infrastructure) and the seeded
input module ``tucker_inputs``; no value here comes from the CUDA path.  The oracle at these sizes
takes minutes on a many-core host, so its results are stored once and the GPU tests compare
against them (the GPU box runs the same image; ``--only cfg5|cfg4|small`` restricts the work).

What is stored per problem (T1–T4 of DESIGN.md §4 need exactly these):
  lam_m      full eigen-spectrum of G_m (descending), the T1 reference and the gap / k_res source
  U_m        the oracle's sign-fixed leading columns, up to the last column whose gap
             (over the full spectrum) is >= 1e-6 lambda_1 — the columns T2 compares
  core_blk   the core's leading block up to k_res(m, 1e-10) per mode (T3)
  core_norm  ||beta||_F of the full core at the stored ranks (T3's norm check)
  E, normF   relative Frobenius error at each listed rank triple (T4)

Problems:
  cfg5  BASELINE config 5: 1024^3 on [-1,1]^3, Matern nu=1.5 ell=0.2 sigma2=1; ranks (40,40,40)
        and its nested truncation (10,10,10) (same eigenvectors, leading core block; SURVEY §8(c)
        "Headline run").  Oracle: orc.hosvd + orc.tucker_error.
  cfg4  BASELINE config 4: 512^3 on [-1,1]^3, the 16 seeded Matern settings (R10), ranks (30,30,30)
        and truncations (10,10,10), (20,20,20).
  small BASELINE configs 1-3 (32^3 nu=1/2 ranks 8; 128^3 closed forms x 9 at ranks 20 with the
        rank sweep 1..20 read as truncations (R11); the anisotropic (256,192,128) grid, general nu
        and Slater, ranks (12,12,10)) — bench.py reports its T1-T4 deltas against these.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from tucker_inputs import config1, config2, config3, config4, config5  # noqa: E402

GAP_REL = 1e-6
KRES_T3 = 1e-10


def gap_ok(lam, k):
    others = np.delete(lam, k)
    return np.min(np.abs(others - lam[k])) >= GAP_REL * lam[0]


def k_res(lam, r, tau):
    return int(np.sum(lam[:r] >= tau * lam[0]))


def solve(grid, kern, r, truncations):
    og = orc.Grid(tuple(grid.n), tuple(grid.lo), tuple(grid.hi))
    ok = orc.Kernel(kern.family, kern.sigma2, kern.ell, kern.nu, kern.lam, kern.p, kern.flags)
    t0 = time.time()
    F = orc.fill(og, ok)
    t1 = time.time()
    h = orc.hosvd(F, r)
    t2 = time.time()
    if h.rc != 0:
        raise RuntimeError(f"oracle hosvd rc={h.rc}")
    out = {"r": np.array(r), "rc": np.array(h.rc)}
    for m in range(3):
        lam = h.lam[m]
        keep = max([c + 1 for c in range(r[m]) if gap_ok(lam, c)] + [0])
        out[f"lam{m}"] = lam
        out[f"U{m}"] = np.ascontiguousarray(h.U[m][:, :keep])
    blk = [k_res(h.lam[m], r[m], KRES_T3) for m in range(3)]
    out["core_blk"] = np.ascontiguousarray(h.core[:blk[0], :blk[1], :blk[2]])
    out["core_norm"] = np.array(np.linalg.norm(h.core))
    Es = []
    for rt in truncations:
        Ut = [np.ascontiguousarray(h.U[m][:, :rt[m]]) for m in range(3)]
        ct = np.ascontiguousarray(h.core[:rt[0], :rt[1], :rt[2]])
        E, nf, nd = orc.tucker_error(F, *Ut, ct)
        Es.append((rt, E, nf, nd))
        out[f"core_norm_r{rt[0]}"] = np.array(np.linalg.norm(ct))
    t3 = time.time()
    out["truncations"] = np.array([e[0] for e in Es])
    out["E"] = np.array([e[1] for e in Es])
    out["normF"] = np.array(Es[0][2])
    out["seconds"] = np.array([t1 - t0, t2 - t1, t3 - t2])
    out["threads"] = np.array(orc.num_threads())
    return out


def kernel_fields(k):
    return np.array([k.family, k.sigma2, k.ell, k.nu, k.lam, k.p, k.flags], dtype=np.float64)


def make_cfg5():
    w = config5((40, 40, 40))
    o = solve(w.grid, w.kernels[0], (40, 40, 40), [(40, 40, 40), (10, 10, 10)])
    o["grid_n"] = np.array(w.grid.n)
    o["kernel"] = kernel_fields(w.kernels[0])
    return o


def make_cfg4(settings):
    w = config4()
    res = {}
    for s in settings:
        k = w.kernels[s]
        o = solve(w.grid, k, (30, 30, 30), [(30, 30, 30), (20, 20, 20), (10, 10, 10)])
        o["kernel"] = kernel_fields(k)
        for key, v in o.items():
            res[f"s{s}_{key}"] = v
        print(f"cfg4 setting {s}: nu={k.nu:.6g} ell={k.ell:.6g} E={o['E']} t={o['seconds']}", flush=True)
    res["settings"] = np.array(settings)
    return res


def make_small():
    res = {}
    for w, truncs in ((config1(), [(8, 8, 8)]),
                      (config2(), [(r, r, r) for r in (20, 15, 10, 5, 1)]),
                      (config3(), [(12, 12, 10)])):
        for i, k in enumerate(w.kernels):
            o = solve(w.grid, k, w.ranks, truncs)
            o["kernel"] = kernel_fields(k)
            o["grid"] = np.array([list(w.grid.n), list(w.grid.lo), list(w.grid.hi)], dtype=np.float64)
            for key, v in o.items():
                res[f"{w.name}_k{i}_{key}"] = v
            print(f"{w.name} kernel {i}: E={o['E']} t={o['seconds']}", flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", choices=["cfg5", "cfg4", "small"], default=None)
    ap.add_argument("--cfg4-settings", default="all")
    ap.add_argument("--out", default=HERE)
    args = ap.parse_args()
    orc.build()
    if args.only in (None, "small"):
        np.savez_compressed(os.path.join(args.out, "small_oracle.npz"), **make_small())
        print("wrote small_oracle.npz", flush=True)
    if args.only in (None, "cfg4"):
        st = list(range(16)) if args.cfg4_settings == "all" else [int(v) for v in args.cfg4_settings.split(",")]
        np.savez_compressed(os.path.join(args.out, "cfg4_512_oracle.npz"), **make_cfg4(st))
        print("wrote cfg4_512_oracle.npz", flush=True)
    if args.only in (None, "cfg5"):
        o = make_cfg5()
        np.savez_compressed(os.path.join(args.out, "cfg5_1024_oracle.npz"), **o)
        print(f"wrote cfg5_1024_oracle.npz: E={o['E']} seconds={o['seconds']} threads={o['threads']}", flush=True)


if __name__ == "__main__":
    main()
