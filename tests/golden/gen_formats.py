#!/usr/bin/env python3
"""Write QSIM / QSCL fixtures with the REFERENCE's own serializers
(tensor_io.hpp:55 serialize_tensor, distill.hpp:296 serialize_scales, via
oracle/_ref/libqfref.so compiled from /root/reference) plus the expected
decoded values, for tests/test_formats.py::test_golden_fixtures_from_reference.

    python tests/golden/gen_formats.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    ref = oracle.Reference()
    rng = np.random.default_rng(2511)
    t = rng.normal(0, 2, (3, 8, 10)).astype(np.float32)
    t.ravel()[:4] = [0.0, -0.0, 65504.0, 1e-45]
    st, blob = ref.serialize_tensor(t, 1)
    assert st == 0
    with open(os.path.join(HERE, "ref_tensor.qsim"), "wb") as f:
        f.write(blob)
    names = ["conv1", "fnet_out", "inet_out", "res1a", "res2_down"]
    scales = {n: (rng.uniform(-7, 0, c).tolist(), float(rng.uniform(-5, -1)))
              for n, c in zip(names, [32, 128, 384, 32, 64])}
    st, sblob = ref.serialize_scales(scales)
    assert st == 0
    with open(os.path.join(HERE, "ref_scales.qscl"), "wb") as f:
        f.write(sblob)
    st, parsed = ref.parse_scales(sblob)
    assert st == 0
    exp = {"tensor_shape": np.array(t.shape, dtype=np.int64), "tensor_prec": np.int64(1),
           "tensor_data": t.ravel(), "scale_names": np.array(list(parsed)),
           "scale_a": np.array([parsed[n][1] for n in parsed])}
    for i, n in enumerate(parsed):
        exp["scale_w_" + str(i)] = np.array(parsed[n][0], dtype=np.float64)
    np.savez(os.path.join(HERE, "formats_expect.npz"), **exp)
    print("wrote", len(blob), "+", len(sblob), "bytes")


if __name__ == "__main__":
    main()
