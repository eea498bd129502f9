"""CPU oracle for the fused fake-quant path — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU reference — never as the thing measured or shipped.

Two CPU implementations are exposed with numpy-array signatures:

* ``Oracle`` — the plain-C restatement (oracle/qf_oracle.c -> liborc.so),
  each function citing the reference file:line it follows.
* ``Reference`` — the UNMODIFIED reference headers compiled from their own
  sources (oracle/Makefile -> oracle/_ref/libqfref.so). Present in the build
  container (built from /root/reference) and shipped prebuilt to the GPU box.

The oracle is pinned against ``Reference`` and the committed golden vectors
under tests/golden/ (see tests/test_oracle_pinning.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libqfref.so")
REF_V3_PATH = os.path.join(HERE, "_ref", "libqfref_v3.so")  # -march=x86-64-v3, timing only

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double
_flt = ctypes.c_float


def build() -> None:
    """Build liborc.so (and _ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class OrcCfg(ctypes.Structure):
    _fields_ = [("bits", _i32), ("reserved", _i32), ("s_min", _dbl), ("s_min_half", _dbl),
                ("s_max", _dbl), ("eps", _dbl)]


def default_cfg(bits: int = 8) -> OrcCfg:
    return OrcCfg(bits, 0, 1e-6, 1e-4, 64.0, 1e-8)


def _ptr_or_null(a):
    return None if a is None else a.ctypes.data_as(_vp)


class Oracle:
    """ctypes view of liborc.so (the C restatement)."""

    def __init__(self, path: str = ORC_PATH):
        if not os.path.exists(path):
            build()
        L = self.L = ctypes.CDLL(path)
        cfgp = ctypes.POINTER(OrcCfg)
        L.orc_softplus.restype = _dbl
        L.orc_softplus.argtypes = [_dbl]
        L.orc_fq_backward_s.restype = _i32
        L.orc_fq_backward_s.argtypes = [_f32p, _f32p, _vp, _i64, _i64, _i64, _f64p, _f64p, _dbl, _f64p]
        L.orc_sigmoid.restype = _dbl
        L.orc_sigmoid.argtypes = [_dbl]
        L.orc_softplus_inv.restype = _i32
        L.orc_softplus_inv.argtypes = [_dbl, ctypes.POINTER(_dbl)]
        L.orc_resolve_scale.restype = _i32
        L.orc_resolve_scale.argtypes = [_dbl, cfgp, _i32, ctypes.POINTER(_dbl)]
        L.orc_cfg_validate.restype = _i32
        L.orc_cfg_validate.argtypes = [cfgp]
        L.orc_f32_to_f16_bits.restype = ctypes.c_uint16
        L.orc_f32_to_f16_bits.argtypes = [_flt]
        L.orc_f16_bits_to_f32.restype = _flt
        L.orc_f16_bits_to_f32.argtypes = [ctypes.c_uint16]
        L.orc_round_to_half.restype = _flt
        L.orc_round_to_half.argtypes = [_flt, ctypes.POINTER(_i32)]
        L.orc_fq_value.restype = _flt
        L.orc_fq_value.argtypes = [_flt, _flt, _flt]
        L.orc_pairwise_sum.restype = _dbl
        L.orc_pairwise_sum.argtypes = [_f64p, _i64]
        L.orc_fake_quantize.restype = _i32
        L.orc_fake_quantize.argtypes = [_f32p, _f32p, _i64, _i64, _i64, _f64p, cfgp, _i32]
        L.orc_fake_quantize_perop.restype = _i32
        L.orc_fake_quantize_perop.argtypes = [_f32p, _f32p, _i64, _i64, _i64, _f64p, cfgp, _i32, _f32p]
        L.orc_int8_codes.restype = _i32
        L.orc_int8_codes.argtypes = [_f32p, _i8p, _i64, _i64, _i64, _f64p, cfgp]
        L.orc_fq_backward.restype = _i32
        L.orc_fq_backward.argtypes = [_f32p, _f32p, _vp, _i64, _i64, _i64, _f64p, cfgp, _i32, _f64p, _i32]
        L.orc_fq_chain.restype = _i32
        L.orc_fq_chain.argtypes = [_f32p, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i32, _i32, cfgp]
        L.orc_gelu.restype = _flt
        L.orc_gelu.argtypes = [_flt]
        L.orc_rng_word.restype = _u64
        L.orc_rng_word.argtypes = [_u64, _u64, _u64]
        L.orc_rng_uniform.restype = _dbl
        L.orc_rng_uniform.argtypes = [_u64, _u64, _u64]
        L.orc_rng_normal.restype = _dbl
        L.orc_rng_normal.argtypes = [_u64, _u64, _u64]
        L.orc_fill_rng.restype = None
        L.orc_fill_rng.argtypes = [_f32p, _i64, _u64, _u64, _u64, _i32, _dbl, _dbl, _i32]
        L.orc_distill_pair.restype = _i32
        L.orc_distill_pair.argtypes = [_f32p, _f32p, _i64, _i64, _dbl, _dbl, _f32p, _f64p]
        L.orc_adam.restype = _i32
        L.orc_adam.argtypes = [_f64p, _f64p, _f64p, _f64p, _i64, _dbl, _dbl, _dbl, _dbl, _i64]

    # scalar math
    def softplus(self, x): return self.L.orc_softplus(x)
    def sigmoid(self, x): return self.L.orc_sigmoid(x)

    def softplus_inv(self, y):
        out = _dbl()
        st = self.L.orc_softplus_inv(y, ctypes.byref(out))
        return st, out.value

    def resolve_scale(self, log_s, half=0, cfg=None):
        out = _dbl()
        st = self.L.orc_resolve_scale(log_s, ctypes.byref(cfg or default_cfg()), half, ctypes.byref(out))
        return st, out.value

    def fq_value(self, x, s, q=127.0): return self.L.orc_fq_value(x, s, q)

    def round_to_half(self, v):
        sat = _i32(0)
        r = self.L.orc_round_to_half(v, ctypes.byref(sat))
        return r, sat.value

    def pairwise_sum(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        return self.L.orc_pairwise_sum(a, a.size)

    # tensor ops on [outer, channels, inner]
    def fake_quantize(self, x, s, outer, channels, inner, half=0, cfg=None):
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        y = np.empty_like(x)
        s = np.ascontiguousarray(s, dtype=np.float64).ravel()
        st = self.L.orc_fake_quantize(x, y, outer, channels, inner, s, ctypes.byref(cfg or default_cfg()), half)
        return st, y

    def fake_quantize_perop(self, x, s, outer, channels, inner, half=0, cfg=None):
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        y = np.empty_like(x)
        tmp = np.empty(3 * x.size, dtype=np.float32)
        s = np.ascontiguousarray(s, dtype=np.float64).ravel()
        st = self.L.orc_fake_quantize_perop(x, y, outer, channels, inner, s,
                                            ctypes.byref(cfg or default_cfg()), half, tmp)
        return st, y

    def int8_codes(self, x, s, outer, channels, inner, cfg=None):
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        c = np.empty(x.size, dtype=np.int8)
        s = np.ascontiguousarray(s, dtype=np.float64).ravel()
        st = self.L.orc_int8_codes(x, c, outer, channels, inner, s, ctypes.byref(cfg or default_cfg()))
        return st, c

    def fq_backward(self, x, up, log_s, outer, channels, inner, half=0, cfg=None,
                    d_log_s=None, accumulate=0, want_dx=True):
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        up = np.ascontiguousarray(up, dtype=np.float32).ravel()
        log_s = np.ascontiguousarray(log_s, dtype=np.float64).ravel()
        dx = np.empty_like(x) if want_dx else None
        dls = (np.zeros(channels, dtype=np.float64) if d_log_s is None
               else np.array(d_log_s, dtype=np.float64).ravel().copy())
        st = self.L.orc_fq_backward(x, up, _ptr_or_null(dx), outer, channels, inner, log_s,
                                    ctypes.byref(cfg or default_cfg()), half, dls, accumulate)
        return st, dx, dls

    def fq_backward_s(self, x, up, s, chain, outer, channels, inner, q=127.0, want_dx=True):
        """fq_backward with the resolved scales and chain factors given."""
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        up = np.ascontiguousarray(up, dtype=np.float32).ravel()
        s = np.ascontiguousarray(s, dtype=np.float64).ravel()
        chain = np.ascontiguousarray(chain, dtype=np.float64).ravel()
        dx = np.empty_like(x) if want_dx else None
        dls = np.zeros(channels, dtype=np.float64)
        st = self.L.orc_fq_backward_s(x, up, _ptr_or_null(dx), outer, channels, inner, s, chain, float(q), dls)
        return st, dx, dls

    def fq_chain(self, a, b, scales, outer, channels, inner, act=1, half=0, preact=False, cfg=None):
        a = np.ascontiguousarray(a, dtype=np.float32).ravel()
        b = None if b is None else np.ascontiguousarray(b, dtype=np.float32).ravel()
        pre = np.empty_like(a) if preact else None
        ys = [np.empty_like(a) for _ in scales]
        ss = [np.ascontiguousarray(s, dtype=np.float64).ravel() for s in scales]
        y0 = ys[0] if len(ys) > 0 else None
        y1 = ys[1] if len(ys) > 1 else None
        s0 = ss[0] if len(ss) > 0 else None
        s1 = ss[1] if len(ss) > 1 else None
        st = self.L.orc_fq_chain(a, _ptr_or_null(b), _ptr_or_null(pre), _ptr_or_null(y0),
                                 _ptr_or_null(y1), _ptr_or_null(s0), _ptr_or_null(s1), outer,
                                 channels, inner, act, half, ctypes.byref(cfg or default_cfg()))
        return st, ys, pre

    def gelu(self, v): return self.L.orc_gelu(v)

    def fill_rng(self, n, seed, stream, kind=1, lo=1.0, hi=0.0, offset=0, half=0):
        out = np.empty(n, dtype=np.float32)
        self.L.orc_fill_rng(out, n, seed, stream, offset, kind, lo, hi, half)
        return out

    def distill_pair(self, s, t, lam, grad_scale=1.0):
        """pair_loss (distill.hpp:66-124) over [C, ...]: (status, [mse, cos], d_s)"""
        s = np.ascontiguousarray(s, dtype=np.float32)
        t = np.ascontiguousarray(t, dtype=np.float32)
        c = s.shape[0]
        hw = s.size // c
        ds = np.zeros_like(s)
        o2 = np.zeros(2, dtype=np.float64)
        st = self.L.orc_distill_pair(s, t, c, hw, lam, grad_scale, ds, o2)
        return st, o2, ds

    def distill_loss(self, fs, ft, is_, it, lam, grad_scale=1.0):
        """distill.hpp:126-141: (status, [total, mse_f, mse_i, cos_f, cos_i], d_f, d_i)"""
        s1, f2, df = self.distill_pair(fs, ft, lam, grad_scale)
        s2, i2, di = self.distill_pair(is_, it, lam, grad_scale)
        total = f2[0] + i2[0] + lam * (1.0 - f2[1]) + lam * (1.0 - i2[1])
        return s1 or s2, np.array([total, f2[0], i2[0], f2[1], i2[1]]), df, di

    def adam(self, p, m, v, g, b1, b2, lr, eps, t):
        """distill.hpp:264-279 in place; returns 1 (skipped) on a non-finite gradient"""
        return self.L.orc_adam(p, m, v, np.ascontiguousarray(g, dtype=np.float64), p.size, b1, b2,
                               lr, eps, t)


class Reference:
    """ctypes view of oracle/_ref/libqfref.so — the reference's own code."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = ctypes.CDLL(path)
        d4 = ctypes.POINTER(_dbl)
        L.ref_softplus.restype = _dbl
        L.ref_softplus.argtypes = [_dbl]
        L.ref_sigmoid.restype = _dbl
        L.ref_sigmoid.argtypes = [_dbl]
        L.ref_softplus_inv.restype = _i32
        L.ref_softplus_inv.argtypes = [_dbl, ctypes.POINTER(_dbl)]
        L.ref_resolve_scale.restype = _i32
        L.ref_resolve_scale.argtypes = [_dbl, _i32, _f64p, _i32, ctypes.POINTER(_dbl)]
        L.ref_cfg_validate.restype = _i32
        L.ref_cfg_validate.argtypes = [_i32, _f64p]
        L.ref_fq_value.restype = _flt
        L.ref_fq_value.argtypes = [_flt, _flt, _flt]
        L.ref_f32_to_f16_bits.restype = ctypes.c_uint16
        L.ref_f32_to_f16_bits.argtypes = [_flt]
        L.ref_f16_bits_to_f32.restype = _flt
        L.ref_f16_bits_to_f32.argtypes = [ctypes.c_uint16]
        L.ref_round_to_half.restype = _flt
        L.ref_round_to_half.argtypes = [_flt, ctypes.POINTER(_i32)]
        L.ref_pairwise_sum.restype = _dbl
        L.ref_pairwise_sum.argtypes = [_f64p, _i64]
        L.ref_fake_quantize.restype = _i32
        L.ref_fake_quantize.argtypes = [_f32p, _i64p, _i32, _i32, _f64p, _i64, _i32, _f64p, _f32p]
        L.ref_fake_quantize_pc.restype = _i32
        L.ref_fake_quantize_pc.argtypes = [_f32p, _i64p, _i32, _i32, _f64p, _i64, _i32, _f64p, _f32p]
        L.ref_int8_codes.restype = _i32
        L.ref_int8_codes.argtypes = [_f32p, _i64p, _i32, _f64p, _i64, _i32, _i32, _f64p, _i8p]
        L.ref_fq_backward.restype = _i32
        L.ref_fq_backward.argtypes = [_f32p, _f32p, _i64p, _i32, _f64p, _i64, _i32, _i32, _i32,
                                      _f64p, _vp, _f64p]
        L.ref_demote_half.restype = _i32
        L.ref_demote_half.argtypes = [_f32p, _i64, _f32p, ctypes.POINTER(_u64)]
        L.ref_residual_join.restype = _i32
        L.ref_residual_join.argtypes = [_f32p, _f32p, _i64, _i32, _f32p]
        L.ref_rng_word.restype = _u64
        L.ref_rng_word.argtypes = [_u64, _u64, _u64]
        L.ref_rng_uniform.restype = _dbl
        L.ref_rng_uniform.argtypes = [_u64, _u64, _u64]
        L.ref_rng_normal.restype = _dbl
        L.ref_rng_normal.argtypes = [_u64, _u64, _u64]
        L.ref_bench_points.restype = _i32
        L.ref_bench_points.argtypes = [_i32, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64p, _i64p,
                                       ctypes.POINTER(_vp), _i32, _i32, _i32, _i32, _i32,
                                       ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)]
        L.ref_bench_sweeps.restype = _i32
        L.ref_bench_sweeps.argtypes = [_i32, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64p, _i64p,
                                       ctypes.POINTER(_vp), _i32, _i32, _i32, _i32,
                                       ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)]

        _sz = ctypes.c_size_t
        L.ref_serialize_tensor.restype = _i32
        L.ref_serialize_tensor.argtypes = [_vp, _vp, _i32, _i32, _vp, _sz, ctypes.POINTER(_sz)]
        L.ref_parse_tensor.restype = _i32
        L.ref_parse_tensor.argtypes = [ctypes.c_char_p, _sz, ctypes.POINTER(_sz), _i64p,
                                       ctypes.POINTER(_i32), ctypes.POINTER(_i32), _vp, _i64,
                                       ctypes.POINTER(_i64)]
        L.ref_serialize_scales.restype = _i32
        L.ref_serialize_scales.argtypes = [_i32, _vp, _vp, _vp, _vp, _vp, _sz, ctypes.POINTER(_sz)]
        L.ref_scales_roundtrip.restype = _i32
        L.ref_scales_roundtrip.argtypes = [ctypes.c_char_p, _sz, _vp, _sz, ctypes.POINTER(_sz)]
        L.ref_scales_layer.restype = _i32
        L.ref_scales_layer.argtypes = [ctypes.c_char_p, _sz, _i32, ctypes.c_char_p, _sz, _f64p, _i64,
                                       ctypes.POINTER(_i64), ctypes.POINTER(_dbl), ctypes.POINTER(_i32)]
        L.ref_distill_loss.restype = _i32
        L.ref_distill_loss.argtypes = [_f32p, _f32p, _i64p, _f32p, _f32p, _i64p, _dbl, _f64p, _f32p,
                                       _f32p]

    # ---- formats (tensor_io.hpp, distill.hpp:287-362) ----
    def serialize_tensor(self, data, precision=0):
        a = np.require(np.asarray(data, dtype=np.float32), requirements='C')
        sh = np.array(a.shape if a.ndim else [], dtype=np.int64)
        size = ctypes.c_size_t()
        shp = sh.ctypes.data if sh.size else None
        st = self.L.ref_serialize_tensor(a.ctypes.data, shp, a.ndim, precision, None, 0, ctypes.byref(size))
        if st:
            return st, None
        out = ctypes.create_string_buffer(size.value)
        st = self.L.ref_serialize_tensor(a.ctypes.data, shp, a.ndim, precision, out, size.value,
                                         ctypes.byref(size))
        return st, out.raw[:size.value]

    def parse_tensor(self, buf, offset=0):
        """-> (status, data, shape, precision, new_offset)"""
        off = ctypes.c_size_t(offset)
        shape = np.zeros(8, dtype=np.int64)
        rank, prec, n = _i32(), _i32(), _i64()
        st = self.L.ref_parse_tensor(buf, len(buf), ctypes.byref(off), shape, ctypes.byref(rank),
                                     ctypes.byref(prec), None, 0, ctypes.byref(n))
        if st:
            return st, None, None, None, offset
        data = np.zeros(max(1, n.value), dtype=np.float32)
        off = ctypes.c_size_t(offset)
        st = self.L.ref_parse_tensor(buf, len(buf), ctypes.byref(off), shape, ctypes.byref(rank),
                                     ctypes.byref(prec), data.ctypes.data, n.value, ctypes.byref(n))
        return st, data[:n.value], tuple(int(v) for v in shape[:rank.value]), prec.value, off.value

    def serialize_scales(self, scales):
        names = list(scales.keys())
        n = len(names)
        enc = [nm.encode("utf-8", "surrogateescape") for nm in names]
        c_names = (ctypes.c_char_p * max(1, n))(*enc)
        ws = [np.ascontiguousarray(np.asarray(scales[nm][0], dtype=np.float64)) for nm in names]
        c_w = (_vp * max(1, n))(*[w.ctypes.data if w.size else None for w in ws])
        c_cnt = (_i64 * max(1, n))(*[w.size for w in ws])
        c_a = (_dbl * max(1, n))(*[float(scales[nm][1]) for nm in names])
        size = ctypes.c_size_t()
        st = self.L.ref_serialize_scales(n, c_names, c_w, c_cnt, c_a, None, 0, ctypes.byref(size))
        if st:
            return st, None
        out = ctypes.create_string_buffer(size.value)
        st = self.L.ref_serialize_scales(n, c_names, c_w, c_cnt, c_a, out, size.value, ctypes.byref(size))
        return st, out.raw[:size.value]

    def scales_roundtrip(self, buf):
        size = ctypes.c_size_t()
        st = self.L.ref_scales_roundtrip(buf, len(buf), None, 0, ctypes.byref(size))
        if st:
            return st, None
        out = ctypes.create_string_buffer(size.value)
        st = self.L.ref_scales_roundtrip(buf, len(buf), out, size.value, ctypes.byref(size))
        return st, out.raw[:size.value]

    def parse_scales(self, buf):
        """-> (status, {name: (log_w list, log_a)})"""
        out = {}
        nl = _i32(0)
        i = 0
        while True:
            name = ctypes.create_string_buffer(4096)
            w = np.zeros(1 << 16, dtype=np.float64)
            cnt, a = _i64(), _dbl()
            st = self.L.ref_scales_layer(buf, len(buf), i, name, 4096, w, w.size, ctypes.byref(cnt),
                                         ctypes.byref(a), ctypes.byref(nl))
            if st:
                return st, None
            if i >= nl.value:
                return 0, out
            out[name.value.decode("utf-8", "surrogateescape")] = (w[:cnt.value].tolist(), a.value)
            i += 1

    def distill_loss(self, fs, ft, is_, it, lam):
        """distill.hpp:126-141 -> (status, [total, mse_f, mse_i, cos_f, cos_i], d_f, d_i)"""
        fs, ft, is_, it = [np.ascontiguousarray(a, dtype=np.float32) for a in (fs, ft, is_, it)]
        fsh = np.array(fs.shape, dtype=np.int64)
        ish = np.array(is_.shape, dtype=np.int64)
        o6 = np.zeros(6, dtype=np.float64)
        df = np.zeros_like(fs)
        di = np.zeros_like(is_)
        st = self.L.ref_distill_loss(fs, ft, fsh, is_, it, ish, lam, o6, df, di)
        return st, o6[:5], df, di

    @staticmethod
    def _d4(cfg=None):
        c = cfg or default_cfg()
        return c.bits, np.array([c.s_min, c.s_min_half, c.s_max, c.eps], dtype=np.float64)

    def softplus(self, x): return self.L.ref_softplus(x)
    def sigmoid(self, x): return self.L.ref_sigmoid(x)

    def softplus_inv(self, y):
        out = _dbl()
        st = self.L.ref_softplus_inv(y, ctypes.byref(out))
        return st, out.value

    def resolve_scale(self, log_s, half=0, cfg=None):
        bits, d4 = self._d4(cfg)
        out = _dbl()
        st = self.L.ref_resolve_scale(log_s, bits, d4, half, ctypes.byref(out))
        return st, out.value

    def cfg_validate(self, cfg):
        bits, d4 = self._d4(cfg)
        return self.L.ref_cfg_validate(bits, d4)

    def fq_value(self, x, s, q=127.0): return self.L.ref_fq_value(x, s, q)

    def round_to_half(self, v):
        sat = _i32(0)
        r = self.L.ref_round_to_half(v, ctypes.byref(sat))
        return r, sat.value

    def pairwise_sum(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        return self.L.ref_pairwise_sum(a, a.size)

    def fake_quantize(self, x, shape, s, half=0, per_channel=None, cfg=None):
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        y = np.empty_like(x)
        s = np.ascontiguousarray(s, dtype=np.float64).ravel()
        shp = np.array(shape, dtype=np.int64)
        bits, d4 = self._d4(cfg)
        fn = self.L.ref_fake_quantize_pc if per_channel else self.L.ref_fake_quantize
        st = fn(x, shp, len(shape), half, s, s.size, bits, d4, y)
        return st, y

    def int8_codes(self, x, shape, s, per_channel=False, cfg=None):
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        c = np.empty(x.size, dtype=np.int8)
        s = np.ascontiguousarray(s, dtype=np.float64).ravel()
        bits, d4 = self._d4(cfg)
        st = self.L.ref_int8_codes(x, np.array(shape, dtype=np.int64), len(shape), s, s.size,
                                   1 if per_channel else 0, bits, d4, c)
        return st, c

    def fq_backward(self, x, up, shape, log_s, per_channel=False, half=0, cfg=None, want_dx=True):
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        up = np.ascontiguousarray(up, dtype=np.float32).ravel()
        log_s = np.ascontiguousarray(log_s, dtype=np.float64).ravel()
        dx = np.empty_like(x) if want_dx else None
        dls = np.zeros(log_s.size, dtype=np.float64)
        bits, d4 = self._d4(cfg)
        st = self.L.ref_fq_backward(x, up, np.array(shape, dtype=np.int64), len(shape), log_s,
                                    log_s.size, 1 if per_channel else 0, half, bits, d4,
                                    _ptr_or_null(dx), dls)
        return st, dx, dls

    def demote_half(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        y = np.empty_like(x)
        ovf = _u64(0)
        st = self.L.ref_demote_half(x, x.size, y, ctypes.byref(ovf))
        return st, y, ovf.value

    def residual_join(self, a, b, half=0):
        a = np.ascontiguousarray(a, dtype=np.float32).ravel()
        b = np.ascontiguousarray(b, dtype=np.float32).ravel()
        y = np.empty_like(a)
        st = self.L.ref_residual_join(a, b, a.size, half, y)
        return st, y

    def bench_points(self, xs, ups, channels, inners, log_ss, half=0, do_fwd=1, do_bwd=1,
                     threads=1, reps=1):
        """Time the reference per-channel FQ fwd + bwd over quant points."""
        n = len(xs)
        arr = lambda lst: (_vp * n)(*[a.ctypes.data_as(_vp) for a in lst])  # noqa: E731
        secs = _dbl()
        cs = _dbl()
        st = self.L.ref_bench_points(n, arr(xs), arr(ups), np.array(channels, dtype=np.int64),
                                     np.array(inners, dtype=np.int64), arr(log_ss), half, do_fwd,
                                     do_bwd, threads, reps, ctypes.byref(secs), ctypes.byref(cs))
        return st, secs.value, cs.value

    def bench_sweeps(self, xs, ups, channels, inners, log_ss, half=0, do_bwd=1, threads=0, reps=1):
        """Time the reference's own schedule: scale pass + Dispatcher sweep
        (exec.hpp:127-146, 248-259, 363-375) + sequential backward per point."""
        n = len(xs)
        arr = lambda lst: (_vp * n)(*[a.ctypes.data_as(_vp) for a in lst])  # noqa: E731
        secs = _dbl()
        cs = _dbl()
        st = self.L.ref_bench_sweeps(n, arr(xs), arr(ups), np.array(channels, dtype=np.int64),
                                     np.array(inners, dtype=np.int64), arr(log_ss), half, do_bwd,
                                     threads, reps, ctypes.byref(secs), ctypes.byref(cs))
        return st, secs.value, cs.value


def reference_available() -> bool:
    return os.path.exists(REF_PATH)
