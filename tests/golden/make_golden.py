"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
reference's proj/core compiled unmodified by oracle/Makefile). Run here, where
/root/reference exists; the fixtures are committed so the GPU box (which has no
/root/reference) can check against them.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (counts, lengths, density name, density kwargs)
CASES = [
    ((8,), (1.0,), "poly", dict(m=1.0, k=1, l=1, n=2)),
    ((12,), (2.0,), "test1d", {}),
    ((4, 6), (1.0, 2.0), "poly", dict(m=0.75, k=1, l=2, n=1)),
    ((6, 4), (1.5, 2.5), "gauss", dict(ell=0.3)),
    ((10, 6), (1.0, 1.0), "matern", dict(nu=1.5, ell=0.1)),
    ((16, 16), (1.0, 1.0), "matern", dict(nu=0.5, ell=0.02)),
    ((2, 4, 6), (1.0, 1.0, 1.0), "aniso", dict(m=1.0, ks=[1, 2, 1], n=2)),
    ((4, 6, 4), (1.0, 2.0, 1.0), "gauss", dict(ell=0.2)),
    ((8, 8, 8), (1.0, 1.0, 1.0), "poly", dict(m=1.0, k=1, l=1, n=2)),
    ((6, 2, 4, 2), (1.0, 1.0, 1.0, 1.0), "constant", dict(c=2.0)),
    ((64, 64), (1.0, 1.0), "gauss", dict(ell=0.05)),
]


def main():
    ref = po.Reference()
    rng = np.random.default_rng(20261019)
    data = {}
    for ci, (counts, lengths, dname, kw) in enumerate(CASES):
        dens = po.density(dname, len(counts), **kw)
        for alg in po.ALGORITHMS:
            nd = ref.count_draws(counts, alg)
            draws = rng.standard_normal(nd)
            field, residue, used = ref.synthesize(counts, lengths, dens, alg, draws)
            assert used == nd
            key = f"c{ci}_a{alg}"
            data[key + "_counts"] = np.array(counts, np.int64)
            data[key + "_lengths"] = np.array(lengths, np.float64)
            data[key + "_family"] = np.array(dens.family)
            data[key + "_r"] = np.array(list(dens.r), np.float64)
            data[key + "_i"] = np.array(list(dens.i), np.int32)
            data[key + "_draws"] = draws
            data[key + "_field"] = field
            data[key + "_residue"] = np.array(residue)
        lin, self_ = ref.conjugate_reps(counts)
        data[f"c{ci}_reps"] = lin
        data[f"c{ci}_reps_self"] = self_
        data[f"c{ci}_cov"] = ref.exact_cov_all(counts, lengths, dens)
    np.savez_compressed(os.path.join(OUT, "reference_fields.npz"), **data)
    print("wrote", len(data), "arrays")


if __name__ == "__main__":
    main()
