"""The oracle against golden vectors produced by the reference itself
(tests/golden/gen_golden.py -> reference_vectors.npz). CPU only; these
fixtures pin the oracle even where /root/reference is absent."""
import os

import numpy as np
import pytest

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz"))


def b32(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def test_fq_and_codes(orc):
    x, s = G["fq_x"], G["fq_s"]
    _, y = orc.fake_quantize(x, s, 1, x.size, 1)
    assert np.array_equal(b32(y), b32(G["fq_y"]))
    _, c = orc.int8_codes(x, s, 1, x.size, 1)
    assert np.array_equal(c, G["fq_codes"])
    _, yh = orc.fake_quantize(G["fqh_x"], [0.0315], 1, 1, G["fqh_x"].size, half=1)
    assert np.array_equal(b32(yh), b32(G["fqh_y"]))


@pytest.mark.parametrize("tag", ["bwd_pt", "bwd_pc"])
def test_backward(orc, tag):
    x, up, ls = G[tag + "_x"], G[tag + "_up"], G[tag + "_ls"]
    C, HW = x.shape
    if tag == "bwd_pt":
        _, dx, dls = orc.fq_backward(x, up, ls, 1, 1, x.size)
    else:
        _, dx, dls = orc.fq_backward(x, up, ls, 1, C, HW)
    assert np.array_equal(b32(dx), b32(G[tag + "_dx"].ravel()))
    assert dls.tobytes() == G[tag + "_dls"].tobytes()


def test_half_pairwise_scale_rng(orc):
    got = np.array([orc.round_to_half(float(v))[0] for v in G["half_in"]], dtype=np.float32)
    assert np.array_equal(b32(got), b32(G["half_out"]))
    off = 0
    for n, want in zip(G["pw_lens"], G["pw_sums"]):
        assert orc.pairwise_sum(G["pw_data"][off:off + n]) == want
        off += n
    for t, s, sh, sg in zip(G["ls"], G["ls_s"], G["ls_sh"], G["ls_sig"]):
        assert orc.resolve_scale(t) == (0, s)
        assert orc.resolve_scale(t, 1) == (0, sh)
        assert orc.sigmoid(t) == sg
    normals = np.array([orc.L.orc_rng_normal(1, 0, i) for i in range(2000)])
    assert normals.tobytes() == G["rng_normal"].tobytes()
    words = np.array([orc.L.orc_rng_word(2024, 3, i) for i in range(2000)], dtype=np.uint64)
    assert np.array_equal(words, G["rng_word"])
