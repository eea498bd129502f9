#!/usr/bin/env python3
"""Distillation-loss vectors from the REFERENCE's qf::distill_loss
(distill.hpp:126-141, oracle/_ref/libqfref.so compiled from
/root/reference) -> tests/golden/distill_vectors.npz, for the oracle (CPU)
and device (GPU box, no reference tree) tests.

    python tests/golden/gen_distill.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    ref = oracle.Reference()
    rng = np.random.default_rng(653)
    cases = [((4, 3, 3), (4, 3, 3), 1.0), ((2, 1, 1), (2, 1, 1), 1.0), ((16, 6, 8), (32, 6, 8), 0.7),
             ((128, 6, 8), (384, 6, 8), 1.0), ((3, 7, 5), (5, 2, 2), 0.0)]
    out = {"n_cases": np.int64(len(cases))}
    for k, (sf, si, lam) in enumerate(cases):
        fs, ft = [rng.normal(0, 1, sf).astype(np.float32) for _ in range(2)]
        is_, it = [rng.normal(0, 1, si).astype(np.float32) for _ in range(2)]
        fs.reshape(sf[0], -1)[:, -1] = 0.0
        if k == 0:
            ft = fs.copy()
        st, o, df, di = ref.distill_loss(fs, ft, is_, it, lam)
        assert st == 0
        out.update({f"fs{k}": fs, f"ft{k}": ft, f"is{k}": is_, f"it{k}": it, f"lam{k}": np.float64(lam),
                    f"out{k}": o, f"df{k}": df, f"di{k}": di})
    np.savez_compressed(os.path.join(HERE, "distill_vectors.npz"), **out)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
