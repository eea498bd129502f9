"""QSIM tensor / QSCL scale formats: libqfb's host
reader/writer (csrc/qfb_formats.cpp) against the reference's own
serialize/parse (tensor_io.hpp:55-125, distill.hpp:287-362) compiled from
its sources (oracle/_ref), plus committed reference-made fixtures
(tests/golden/*.qsim|qscl, made by tests/golden/gen_golden.py) that travel
without /root/reference. CPU only."""
import os

import numpy as np
import pytest

import paper_2511_12653_b200 as q
from paper_2511_12653_b200 import formats as F

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


SHAPES = [(), (1,), (7,), (2, 3, 4), (3, 1, 5, 2), (128, 12, 16)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("prec", [0, 1])
def test_tensor_bytes_identical_to_reference(ref, shape, prec):
    rng = np.random.default_rng(len(shape) * 10 + prec)
    a = rng.normal(0, 3, shape).astype(np.float32)
    if a.size:
        a.ravel()[0] = -0.0
        a.ravel()[-1] = np.float32(np.nan) if a.size > 2 else a.ravel()[-1]
    st, want = ref.serialize_tensor(a, prec)
    assert st == 0
    got = F.serialize_tensor(a, prec)
    assert got == want
    t, off = F.parse_tensor(want)
    assert off == len(want) and t.shape == tuple(shape) and t.precision == prec
    assert np.array_equal(bits(t.data.ravel()), bits(a.ravel()))


def test_tensor_blob_of_several_and_offsets(ref):
    rng = np.random.default_rng(3)
    parts = [rng.normal(0, 1, s).astype(np.float32) for s in [(4,), (2, 3), (5, 1, 2)]]
    blob = b"".join(F.serialize_tensor(p) for p in parts)
    off = 0
    for p in parts:
        st, data, shape, prec, roff = ref.parse_tensor(blob, off)
        t, off2 = F.parse_tensor(blob, off)
        assert st == 0 and roff == off2 and shape == t.shape
        assert np.array_equal(bits(t.data.ravel()), bits(data))
        off = off2
    assert off == len(blob)


def test_tensor_errors_match_reference(ref):
    good = F.serialize_tensor(np.arange(6, dtype=np.float32).reshape(2, 3))
    bad_magic = b"X" + good[1:]
    bad_ver = good[:4] + (2).to_bytes(4, "little") + good[8:]
    for blob in [bad_magic, bad_ver] + [good[:k] for k in range(len(good))]:
        st = ref.parse_tensor(blob)[0]
        assert st == 3, (blob, st)           # qf::IoError
        with pytest.raises(q.IoError):
            F.parse_tensor(blob)
    with pytest.raises(q.IoError, match="bad tensor magic"):
        F.parse_tensor(bad_magic)
    with pytest.raises(q.IoError, match="unsupported tensor format version 2"):
        F.parse_tensor(bad_ver)


def test_tensor_nonpositive_dims_are_shape_errors():
    """qf::Tensor rejects dims <= 0 (tensor.hpp:66-73): serialize refuses
    them and a blob carrying one is a ShapeError, not a tensor."""
    with pytest.raises(q.ShapeError):
        F.serialize_tensor(np.zeros((2, 3), np.float32), shape=(2, 0, 3))
    good = F.serialize_tensor(np.zeros((2, 3), np.float32))
    zero = good[:12] + (0).to_bytes(8, "little") + good[20:]
    with pytest.raises(q.ShapeError):
        F.parse_tensor(zero)


def test_tensor_file_roundtrip(tmp_path):
    a = np.random.default_rng(1).normal(0, 1, (3, 4, 5)).astype(np.float32)
    p = str(tmp_path / "t.qsim")
    F.save_tensor(p, a, F.PREC_HALF)
    t = F.load_tensor(p)
    assert t.precision == F.PREC_HALF and np.array_equal(bits(t.data), bits(a))
    with open(p, "ab") as f:
        f.write(b"\0")
    with pytest.raises(q.IoError, match="trailing bytes"):
        F.load_tensor(p)
    with pytest.raises(q.IoError, match="cannot open"):
        F.load_tensor(str(tmp_path / "missing.qsim"))


def scale_set(seed, names=None):
    rng = np.random.default_rng(seed)
    names = names or ["conv1", "res1a", "res1b", "res2_down", "fnet_out", "inet_out"]
    return {n: (rng.uniform(-6, 1, int(rng.integers(0, 40))).tolist(), float(rng.uniform(-5, 0)))
            for n in names}


NAMES = [None, ["a"], [], ['quo"te', "back\\slash", "tab\there", "nl\nx", "ctl\x01", "utf8-é漢"],
         ["z", "a", "m", "A", "_"]]


@pytest.mark.parametrize("names", NAMES)
def test_scales_bytes_identical_to_reference(ref, names):
    s = scale_set(len(names or []) + 1, names)
    st, want = ref.serialize_scales(s)
    assert st == 0
    got = F.serialize_scales(s)
    assert got == want
    st, rt = ref.scales_roundtrip(got)      # save -> load -> save (test_distill.cpp:189-196)
    assert st == 0 and rt == got
    mine = F.parse_scales(want)
    st, theirs = ref.parse_scales(want)
    assert st == 0 and list(mine) == list(theirs)
    for k in mine:
        assert np.array_equal(np.array(mine[k][0]), np.array(theirs[k][0])) and mine[k][1] == theirs[k][1]
        # stored as float32 (distill.hpp:305-308)
        assert np.array_equal(np.array(mine[k][0]), np.array(s[k][0], dtype=np.float32).astype(np.float64))


def test_scales_parse_is_json_general(ref):
    """Whitespace, key order, escapes and duplicate keys read like nlohmann::json."""
    payload = np.array([0.5, -1.25, 2.0], dtype=np.float32).tobytes()
    man = ('{ "layers" : { "b\\u00e9" : {"log_a_off": 8, "log_w_count": 2, "log_w_off": 0},\n'
           '  "a" : {"log_w_off":8,"log_w_count":1,"log_a_off":0,"log_a_off":4} }, "version": 1 }')
    blob = b"QSCL" + (1).to_bytes(4, "little") + len(man.encode()).to_bytes(8, "little") + man.encode() + payload
    mine = F.parse_scales(blob)
    st, theirs = ref.parse_scales(blob)
    assert st == 0 and mine == theirs
    assert list(mine) == ["a", "bé"]


def test_scales_errors_match_reference(ref):
    good = F.serialize_scales(scale_set(5))
    bad = bytearray(good)
    bad[2] = ord("X")   # test_distill.cpp:202-204
    cases = [bytes(bad), good[:4] + (9).to_bytes(4, "little") + good[8:],
             good[:8] + (1 << 40).to_bytes(8, "little") + good[16:],
             good[:16] + b"[" + good[17:],
             good[:-1]]
    cases += [good[:k] for k in range(0, len(good), 7)]
    for blob in cases:
        st = ref.parse_scales(blob)[0]
        assert st != 0, blob
        with pytest.raises(q.IoError):
            F.parse_scales(blob)
    with pytest.raises(q.IoError, match="bad scales magic"):
        F.parse_scales(bytes(bad))
    with pytest.raises(q.IoError, match="unsupported scales version 9"):
        F.parse_scales(cases[1])
    with pytest.raises(q.IoError, match="scales payload truncated"):
        F.parse_scales(good[:-1])


def test_golden_fixtures_from_reference(tmp_path):
    """Files written by the reference itself (travel to the GPU box)."""
    g = np.load(os.path.join(GOLD, "formats_expect.npz"))
    t = F.load_tensor(os.path.join(GOLD, "ref_tensor.qsim"))
    assert t.shape == tuple(g["tensor_shape"]) and t.precision == int(g["tensor_prec"])
    assert np.array_equal(bits(t.data.ravel()), bits(g["tensor_data"]))
    s = F.load_scales(os.path.join(GOLD, "ref_scales.qscl"))
    names = [str(n) for n in g["scale_names"]]
    assert list(s) == names
    for i, n in enumerate(names):
        w = g["scale_w_" + str(i)]
        assert np.array_equal(np.array(s[n][0]), w) and s[n][1] == g["scale_a"][i]
    # our writer reproduces the reference's bytes
    with open(os.path.join(GOLD, "ref_scales.qscl"), "rb") as f:
        assert F.serialize_scales(s) == f.read()
    with open(os.path.join(GOLD, "ref_tensor.qsim"), "rb") as f:
        assert F.serialize_tensor(t.data, t.precision) == f.read()
