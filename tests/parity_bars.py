"""The T1–T4 parity bars of DESIGN.md §4 (BASELINE.json north_star tolerances, reading R14), applied
to a GPU HOSVD result against an oracle reference.  Test code only: the reference is either a live
oracle run (``orc.hosvd``) or a golden file written by ``tests/golden/make_golden.py`` (oracle only).

  T1  |lambda_g - lambda_o| <= 1e-11 lambda_o + 1e-14 lambda_o1         (eigenvalues, lambda = sigma^2)
  T2  max|u_g - u_o| <= 1e-9 on columns with gap >= 1e-6 lambda_1        (gap over the full spectrum)
  T2' ||U^T U - I||_max <= 1e-12
  T3  ||beta_g - beta_o|| <= 1e-10 ||beta_o|| on the block k_res(., 1e-10);  | ||beta_g|| - ||beta_o|| |
      <= 1e-12 ||beta_o||
  T4  |E_g - E_o| <= 1e-12 if every r_m <= k_res(m, 1e-12), else <= max(1e-12, 1e-15 / E_o)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def gap_ok(lam_full, k, rel=1e-6):
    others = np.delete(lam_full, k)
    return np.min(np.abs(others - lam_full[k])) >= rel * lam_full[0]


def k_res(lam, r, tau):
    return int(np.sum(lam[:r] >= tau * lam[0]))


@dataclass
class Ref:
    """Oracle reference of one HOSVD: full spectra, sign-fixed columns (at least the gap-separated
    leading ones), the core's leading block, the full core norm at these ranks and E."""
    lam: list
    U: list
    core_blk: np.ndarray
    core_norm: float
    E: float
    normF: float = float("nan")

    @staticmethod
    def from_oracle(h, E, normF=float("nan")):
        return Ref(list(h.lam), list(h.U), h.core, float(np.linalg.norm(h.core)), float(E), float(normF))


@dataclass
class Deltas:
    """Worst observed deviations (reported by bench.py and the tests), each with its bar."""
    t1: float = 0.0          # max |dlambda| / (1e-11 lambda + 1e-14 lambda_1)  (<= 1 passes)
    t2: float = 0.0          # max column difference over the gap-separated columns
    t2p: float = 0.0         # ||U^T U - I||_max
    t3: float = 0.0          # relative core difference on the resolved block
    t3n: float = 0.0         # relative core-norm difference
    t4: float = 0.0          # |E_g - E_o|
    t4_bar: float = 1e-12
    resolved: bool = True
    columns_checked: list = field(default_factory=list)

    def as_dict(self):
        return {"T1_ratio": self.t1, "T2_max_col": self.t2, "T2p_orth": self.t2p, "T3_rel": self.t3,
                "T3_norm_rel": self.t3n, "T4_abs": self.t4, "T4_bar": self.t4_bar, "resolved": self.resolved,
                "T2_columns": self.columns_checked}


def compare(ref: Ref, r, sigma, U, core, E, check=True, tau4=1e-12) -> Deltas:
    """Apply T1-T4.  sigma, U: lists of numpy arrays (GPU result); core numpy; E float.
    tau4: the resolved threshold of T4 (1e-12; 1e-11 for the DMMA Gram engine, whose FP64
    accumulation over K = n^2 terms adds ~sqrt(K) eps lambda_1 of noise — SURVEY §8(c) T4, DESIGN R19)."""
    d = Deltas()
    blocks = []
    for m in range(3):
        lam_o = np.asarray(ref.lam[m])
        rr = int(r[m])
        lam_g = np.asarray(sigma[m])[:rr] ** 2
        pos = lam_o[:rr] > 0
        bar = 1e-11 * lam_o[:rr][pos] + 1e-14 * lam_o[0]
        d.t1 = max(d.t1, float(np.max(np.abs(lam_g[pos] - lam_o[:rr][pos]) / bar)) if pos.any() else 0.0)
        Ug = np.asarray(U[m])
        Uo = np.asarray(ref.U[m])
        cols = [c for c in range(rr) if gap_ok(lam_o, c)]
        for c in cols:
            assert c < Uo.shape[1], "reference lacks a gap-separated column"
            d.t2 = max(d.t2, float(np.max(np.abs(Ug[:, c] - Uo[:, c]))))
        d.columns_checked.append(len(cols))
        d.t2p = max(d.t2p, float(np.max(np.abs(Ug[:, :rr].T @ Ug[:, :rr] - np.eye(rr)))))
        d.resolved &= rr <= k_res(lam_o, rr, tau4)
        blocks.append(k_res(lam_o, rr, 1e-10))
    a, b, c = blocks
    co = np.asarray(ref.core_blk)[:a, :b, :c]
    cg = np.asarray(core)[:a, :b, :c]
    d.t3 = float(np.linalg.norm(cg - co) / np.linalg.norm(co))
    d.t3n = float(abs(np.linalg.norm(np.asarray(core)) - ref.core_norm) / ref.core_norm)
    d.t4 = float(abs(E - ref.E))
    d.t4_bar = 1e-12 if d.resolved else max(1e-12, 1e-15 / ref.E)
    if check:
        assert d.t1 <= 1.0, ("T1", d.as_dict())
        assert d.t2 <= 1e-9, ("T2", d.as_dict())
        assert d.t2p <= 1e-12, ("T2'", d.as_dict())
        assert d.t3 <= 1e-10, ("T3", d.as_dict())
        assert d.t3n <= 1e-12, ("T3 norm", d.as_dict())
        assert d.t4 <= d.t4_bar, ("T4", d.as_dict(), E, ref.E)
    return d


def golden_ref(z, prefix="", trunc=None) -> Ref:
    """Ref from a make_golden.py npz (``prefix`` selects a config-4 setting, e.g. "s3_").  ``trunc``
    = a rank triple of the stored truncations: its E and core norm (the columns and the core block
    are the leading ones of the stored ranks, the same numbers at any truncation)."""
    g = lambda k: z[prefix + k]  # noqa: E731
    tr = [tuple(int(v) for v in t) for t in g("truncations")]
    ti = 0 if trunc is None else tr.index(tuple(trunc))
    core_norm = float(g("core_norm")) if ti == 0 else float(g(f"core_norm_r{tr[ti][0]}"))
    return Ref([g(f"lam{m}") for m in range(3)], [g(f"U{m}") for m in range(3)], g("core_blk"), core_norm,
               float(g("E")[ti]), float(g("normF")))


def i8_bound_entry(maxabs_a, maxabs_b, l1_a, l1_b, K, b, G_ab, eps=np.finfo(np.float64).eps):
    """R18's element bound of the INT8-emulated Gram for one entry: rows scaled by 2^(b - E_i) with
    max|a_i| < 2^E_i and rounded (error <= 2^(E_i - b - 1) per entry), S formed exactly, one
    rounding — |dG_ab| <= 2^(E_a-b-1)||a_b||_1 + 2^(E_b-b-1)||a_a||_1 + 3 2^(E_a+E_b-2b-2) K + eps|G_ab|
    (+ the reference's own Dot2 error, a few eps|G_ab|)."""
    Ea = np.frexp(maxabs_a)[1] if maxabs_a > 0 else 0
    Eb = np.frexp(maxabs_b)[1] if maxabs_b > 0 else 0
    sa, sb = np.exp2(Ea - b - 1), np.exp2(Eb - b - 1)
    return sa * l1_b + sb * l1_a + 3.0 * sa * sb * K + 4.0 * eps * abs(G_ab)
