"""The reference's on-disk formats through the C-ABI.

QSIM tensors (tensor_io.hpp:1-125) and QSCL scale checkpoints
(distill.hpp:287-362), read and written by libqfb's host code
(csrc/qfb_formats.cpp) byte-for-byte like the reference, so tensors and
scales produced by the reference tools feed the GPU path (load ->
torch.from_numpy(...).cuda()) and our results go back to them.

    t = load_tensor("x.qsim")          # TensorFile(data, shape, precision)
    save_tensor("y.qsim", array, precision=PREC_FULL)
    scales = load_scales("s.qscl")     # {layer: (log_w list, log_a)}
    save_scales("s2.qscl", scales)

Errors raise the package's IoError (qf::IoError) with the reference's
messages.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import _lib, check

_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("qfb_qsim_parse", _i32, [_vp, _sz, ctypes.POINTER(_sz), ctypes.POINTER(_vp)])
_sig("qfb_qsim_load", _i32, [ctypes.c_char_p, ctypes.POINTER(_vp)])
_sig("qfb_qsim_info", _i32, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(ctypes.POINTER(_i64)),
                             ctypes.POINTER(_i32), ctypes.POINTER(_i64),
                             ctypes.POINTER(ctypes.POINTER(ctypes.c_float))])
_sig("qfb_qsim_free", None, [_vp])
_sig("qfb_qsim_serialize", _i32, [_vp, _i32, _vp, _i32, _vp, _sz, ctypes.POINTER(_sz)])
_sig("qfb_qsim_save", _i32, [ctypes.c_char_p, _vp, _i32, _vp, _i32])
_sig("qfb_qscl_parse", _i32, [_vp, _sz, ctypes.POINTER(_vp)])
_sig("qfb_qscl_load", _i32, [ctypes.c_char_p, ctypes.POINTER(_vp)])
_sig("qfb_qscl_count", _i32, [_vp])
_sig("qfb_qscl_layer", _i32, [_vp, _i32, ctypes.POINTER(ctypes.c_char_p),
                              ctypes.POINTER(ctypes.POINTER(ctypes.c_double)), ctypes.POINTER(_i64),
                              ctypes.POINTER(ctypes.c_double)])
_sig("qfb_qscl_free", None, [_vp])
_sig("qfb_qscl_serialize", _i32, [_i32, _vp, _vp, _vp, _vp, _vp, _sz, ctypes.POINTER(_sz)])
_sig("qfb_qscl_save", _i32, [ctypes.c_char_p, _i32, _vp, _vp, _vp, _vp])

PREC_FULL, PREC_HALF = 0, 1   # qf::Precision tag byte (tensor.hpp:25)


@dataclass
class TensorFile:
    data: np.ndarray          # float32, shaped
    shape: Tuple[int, ...]
    precision: int


def _take_tensor(h) -> TensorFile:
    rank, prec, n = _i32(), _i32(), _i64()
    shp = ctypes.POINTER(_i64)()
    dat = ctypes.POINTER(ctypes.c_float)()
    try:
        check(_lib.qfb_qsim_info(h, ctypes.byref(rank), ctypes.byref(shp), ctypes.byref(prec),
                                 ctypes.byref(n), ctypes.byref(dat)))
        shape = tuple(int(shp[i]) for i in range(rank.value))
        data = (np.ctypeslib.as_array(dat, shape=(n.value,)).copy() if n.value
                else np.zeros(0, dtype=np.float32))
        return TensorFile(data.reshape(shape), shape, int(prec.value))
    finally:
        _lib.qfb_qsim_free(h)


def parse_tensor(buf: bytes, offset: int = 0) -> Tuple[TensorFile, int]:
    """qf::parse_tensor (tensor_io.hpp:68): one tensor at `offset`; returns
    it and the offset just past it."""
    off = _sz(offset)
    h = _vp()
    check(_lib.qfb_qsim_parse(buf, len(buf), ctypes.byref(off), ctypes.byref(h)))
    return _take_tensor(h), int(off.value)


def load_tensor(path: str) -> TensorFile:
    """qf::load_tensor (tensor_io.hpp:119): exactly one tensor per file."""
    h = _vp()
    check(_lib.qfb_qsim_load(path.encode(), ctypes.byref(h)))
    return _take_tensor(h)


def _shape_arr(shape: Sequence[int]):
    return (_i64 * max(1, len(shape)))(*shape)


def serialize_tensor(data, precision: int = PREC_FULL, shape: Sequence[int] = None) -> bytes:
    """qf::serialize_tensor (tensor_io.hpp:55), byte-identical."""
    a = np.require(np.asarray(data, dtype=np.float32), requirements='C')
    shape = tuple(a.shape) if shape is None else tuple(shape)
    size = _sz()
    check(_lib.qfb_qsim_serialize(a.ctypes.data, len(shape), _shape_arr(shape), precision, None, 0,
                                  ctypes.byref(size)))
    out = ctypes.create_string_buffer(size.value)
    check(_lib.qfb_qsim_serialize(a.ctypes.data, len(shape), _shape_arr(shape), precision, out,
                                  size.value, ctypes.byref(size)))
    return out.raw[:size.value]


def save_tensor(path: str, data, precision: int = PREC_FULL) -> None:
    """qf::save_tensor (tensor_io.hpp:115)."""
    a = np.require(np.asarray(data, dtype=np.float32), requirements='C')
    check(_lib.qfb_qsim_save(path.encode(), a.ctypes.data, a.ndim, _shape_arr(a.shape), precision))


ScaleSet = Dict[str, Tuple[List[float], float]]


def _take_scales(h) -> ScaleSet:
    out: ScaleSet = {}
    try:
        for i in range(_lib.qfb_qscl_count(h)):
            name = ctypes.c_char_p()
            w = ctypes.POINTER(ctypes.c_double)()
            cnt = _i64()
            a = ctypes.c_double()
            check(_lib.qfb_qscl_layer(h, i, ctypes.byref(name), ctypes.byref(w), ctypes.byref(cnt),
                                      ctypes.byref(a)))
            out[name.value.decode("utf-8", "surrogateescape")] = ([w[k] for k in range(cnt.value)], a.value)
    finally:
        _lib.qfb_qscl_free(h)
    return out


def parse_scales(buf: bytes) -> ScaleSet:
    """qf::parse_scales (distill.hpp:324): {layer: (log_w_scale, log_a_scale)}
    in name order; values are the stored float32 widened to double."""
    h = _vp()
    check(_lib.qfb_qscl_parse(buf, len(buf), ctypes.byref(h)))
    return _take_scales(h)


def load_scales(path: str) -> ScaleSet:
    """qf::load_scales (distill.hpp:360)."""
    h = _vp()
    check(_lib.qfb_qscl_load(path.encode(), ctypes.byref(h)))
    return _take_scales(h)


def _scale_args(scales: ScaleSet):
    names = list(scales.keys())
    n = len(names)
    enc = [nm.encode("utf-8", "surrogateescape") for nm in names]
    c_names = (ctypes.c_char_p * max(1, n))(*enc)
    ws = [np.ascontiguousarray(np.asarray(scales[nm][0], dtype=np.float64)) for nm in names]
    c_w = (_vp * max(1, n))(*[w.ctypes.data if w.size else None for w in ws])
    c_cnt = (_i64 * max(1, n))(*[w.size for w in ws])
    c_a = (ctypes.c_double * max(1, n))(*[float(scales[nm][1]) for nm in names])
    return n, c_names, c_w, c_cnt, c_a, ws


def serialize_scales(scales: ScaleSet) -> bytes:
    """qf::serialize_scales (distill.hpp:296), byte-identical."""
    n, c_names, c_w, c_cnt, c_a, _keep = _scale_args(scales)
    size = _sz()
    check(_lib.qfb_qscl_serialize(n, c_names, c_w, c_cnt, c_a, None, 0, ctypes.byref(size)))
    out = ctypes.create_string_buffer(size.value)
    check(_lib.qfb_qscl_serialize(n, c_names, c_w, c_cnt, c_a, out, size.value, ctypes.byref(size)))
    return out.raw[:size.value]


def save_scales(path: str, scales: ScaleSet) -> None:
    """qf::save_scales (distill.hpp:320)."""
    n, c_names, c_w, c_cnt, c_a, _keep = _scale_args(scales)
    check(_lib.qfb_qscl_save(path.encode(), n, c_names, c_w, c_cnt, c_a))
