"""paper_2511_12653_b200._api — the ctypes binding of libqfb.so (include/qfb.h).

Loaded on first use of any package attribute (see ``__init__``): importing
the package, or a pure-Python submodule such as ``shapes``, maps no native
code. A missing library raises ImportError at that first use — there is no
CPU or eager-PyTorch fallback.
"""
from __future__ import annotations

import builtins
import ctypes
import dataclasses
import os
from typing import Optional, Sequence, Union

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QFB_LIB_PATH") or os.path.join(_HERE, "libqfb.so")  # override: tuning builds

# ---------------------------------------------------------------- errors --


class QfError(RuntimeError):
    """Base of the qf error taxonomy."""


class ShapeError(QfError):
    """qf::ShapeError (errors.hpp:11)."""


class ValueError(QfError, builtins.ValueError):  # noqa: A001 - mirrors qf::ValueError
    """qf::ValueError (errors.hpp:16)."""


class IoError(QfError):
    """qf::IoError (errors.hpp:21)."""


class NonFiniteError(QfError):
    """qf::NonFiniteError (errors.hpp:26)."""


class InsufficientMatchesError(QfError):
    """qf::InsufficientMatchesError (errors.hpp:31)."""


class FusedPathError(QfError):
    """qf::FusedPathError (exec.hpp:51)."""


class CudaError(QfError):
    pass


class NcclError(QfError):
    pass


class UnsupportedError(QfError):
    pass


_STATUS = {
    1: ShapeError,
    2: ValueError,
    3: IoError,
    4: NonFiniteError,
    5: InsufficientMatchesError,
    6: FusedPathError,
    7: CudaError,
    8: NcclError,
    9: UnsupportedError,
}

F32, F16 = 0, 1
PREC_FULL, PREC_HALF = 0, 1
FLAG_HALF_GRID, FLAG_STREAMING = 0x1, 0x2
BWD_ROWS = 2  # qfb_bwd_desc.accumulate: one scale-gradient row per outer index
ACT_NONE, ACT_RELU, ACT_GELU = 0, 1, 2

# ------------------------------------------------------------ library --

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libqfb.so not found at {LIB_PATH}: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        " (there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_u32 = ctypes.c_uint32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double
_pd = ctypes.POINTER(ctypes.c_double)
_pf = ctypes.POINTER(ctypes.c_float)


class CQuantConfig(ctypes.Structure):
    _fields_ = [("bits", _i32), ("reserved", _i32), ("s_min", _dbl), ("s_min_half", _dbl),
                ("s_max", _dbl), ("eps", _dbl)]


class CFqDesc(ctypes.Structure):
    _fields_ = [("x", _vp), ("y", _vp * 2), ("scale", _vp * 2), ("outer", _i64),
                ("channels", _i64), ("inner", _i64), ("n_out", _i32), ("q_max", _i32),
                ("flags", _u32), ("reserved", _u32)]


class CBwdDesc(ctypes.Structure):
    _fields_ = [("x", _vp), ("up", _vp), ("dx", _vp), ("scale64", _vp), ("chain", _vp),
                ("d_log_s", _vp), ("outer", _i64), ("channels", _i64), ("inner", _i64),
                ("q_max", _i32), ("accumulate", _i32), ("row_stride", _i64)]


class CChainDesc(ctypes.Structure):
    _fields_ = [("a", _vp), ("b", _vp), ("preact", _vp), ("y", _vp * 2), ("scale", _vp * 2),
                ("outer", _i64), ("channels", _i64), ("inner", _i64), ("n_out", _i32),
                ("act", _i32), ("dtype", _i32), ("q_max", _i32), ("flags", _u32),
                ("reserved", _u32)]


class CHostPoint(ctypes.Structure):
    _fields_ = [("x", _vp), ("outer", _i64), ("channels", _i64), ("inner", _i64),
                ("n_out", _i32), ("reserved", _i32), ("s", _vp * 2), ("y", _vp * 2),
                ("log_s", _vp * 2), ("up", _vp * 2), ("dx", _vp * 2), ("d_log_s", _vp * 2)]


class CExecPlan(ctypes.Structure):
    _fields_ = [("mode", _i32), ("policy", _i32), ("fallback_enabled", _i32),
                ("cache_weights", _i32), ("fault_inject_layer", _i32), ("reserved", _i32)]


class CExecTrace(ctypes.Structure):
    _fields_ = [("pass_count", _i64), ("bytes_read", _i64), ("bytes_written", _i64),
                ("launches", _i64), ("peak_scratch_bytes", _i64), ("fell_back", _i32),
                ("layers", _i32)]


class CQuantLayer(ctypes.Structure):
    _fields_ = [("index", _i32), ("reserved", _i32), ("weight", _vp), ("c_out", _i64),
                ("per", _i64), ("log_w", _vp), ("log_a", _dbl)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_lib.qfb_last_error.restype = ctypes.c_char_p
_lib.qfb_status_name.restype = ctypes.c_char_p
_lib.qfb_build_info.restype = ctypes.c_char_p
_sig("qfb_quant_config_default", None, [ctypes.POINTER(CQuantConfig)])
_sig("qfb_quant_config_validate", _i32, [ctypes.POINTER(CQuantConfig)])
_sig("qfb_q_max", _i32, [ctypes.POINTER(CQuantConfig)])
_sig("qfb_softplus", _dbl, [_dbl])
_sig("qfb_sigmoid", _dbl, [_dbl])
_sig("qfb_softplus_inv", _i32, [_dbl, _pd])
_sig("qfb_resolve_scales", _i32, [_pd, _i64, ctypes.POINTER(CQuantConfig), _i32, _pd])
_sig("qfb_scale_grad_factors", _i32, [_pd, _i64, ctypes.POINTER(CQuantConfig), _i32, _pd, _pd])
_sig("qfb_cast_scales_f32", _i32, [_pd, _i64, _pf])
_sig("qfb_ctx_create", _i32, [_i32, _vp, ctypes.POINTER(_vp)])
_sig("qfb_ctx_destroy", _i32, [_vp])
_sig("qfb_ctx_set_stream", _i32, [_vp, _vp])
_sig("qfb_ctx_set_option", _i32, [_vp, _i32, _i64])
OPT_BWD_HALF_FP32 = 1  # QFB_OPT_BWD_HALF_FP32
OPT_MAIN_PASS_EVENT = 2  # QFB_OPT_MAIN_PASS_EVENT (profiling hook)
OPT_BWD_ASYNC_FINISH = 3  # QFB_OPT_BWD_ASYNC_FINISH
_sig("qfb_ctx_join", _i32, [_vp])
_sig("qfb_ctx_stream", _vp, [_vp])
_sig("qfb_ctx_sm_count", _i32, [_vp])
_sig("qfb_ctx_sync", _i32, [_vp])
_sig("qfb_ctx_launch_count", _i64, [_vp])
_sig("qfb_fq_fwd", _i32, [_vp, _i32, _vp, _vp, _i64, _i64, _i64, _vp, _i32, _u32])
_sig("qfb_int8_codes", _i32, [_vp, _i32, _vp, _vp, _i64, _i64, _i64, _vp, _i32])
_sig("qfb_fq_bwd", _i32, [_vp, _i32, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _i32, _vp, _i32])
_sig("qfb_fq_chain", _i32, [_vp, ctypes.POINTER(CChainDesc)])
_sig("qfb_fq_chain_multi", _i32, [_vp, ctypes.POINTER(CChainDesc), _i32])
_sig("qfb_fq_fwd_multi", _i32, [_vp, _i32, ctypes.POINTER(CFqDesc), _i32])
_sig("qfb_fq_bwd_multi", _i32, [_vp, _i32, ctypes.POINTER(CBwdDesc), _i32])
_sig("qfb_fq_bwd_reserve", _i32, [_vp, _i32, ctypes.POINTER(CBwdDesc), _i32])
_sig("qfb_resolve_scales_dev", _i32, [_vp, _vp, _i64, ctypes.POINTER(CQuantConfig), _i32, _vp, _vp, _vp])
_sig("qfb_fill_rng", _i32, [_vp, _i32, _vp, _i64, _u64, _u64, _u64, _i32, _dbl, _dbl])
_sig("qfb_fq_fwd_perop", _i32, [_vp, _i32, _vp, _vp, _i64, _i64, _i64, _vp, _i32, _u32, _vp])
_sig("qfb_fake_quantize_host", _i32, [_vp, _i32, _vp, _vp, _i64, _i64, _i64, _pd, ctypes.POINTER(CQuantConfig)])
_sig("qfb_int8_codes_host", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, _pd, ctypes.POINTER(CQuantConfig)])
_sig("qfb_exec_create", _i32, [_vp, ctypes.POINTER(CExecPlan), ctypes.POINTER(_vp)])
_sig("qfb_exec_destroy", _i32, [_vp])
_sig("qfb_exec_quant_layer", _i32, [_vp, ctypes.POINTER(CQuantLayer), ctypes.POINTER(CQuantConfig), _i32,
                                    _vp, _i64, _vp, _vp, ctypes.POINTER(_vp)])
_sig("qfb_exec_trace_get", _i32, [_vp, ctypes.POINTER(CExecTrace)])
_sig("qfb_exec_trace_reset", _i32, [_vp])
_sig("qfb_exec_model_layer", _i32, [ctypes.POINTER(CExecPlan), _i64, _i64, _i64, _i32, _i32,
                                    ctypes.POINTER(CExecTrace)])
_sig("qfb_quant_pass_host", _i32, [_vp, _i32, ctypes.POINTER(CHostPoint), _i32, ctypes.POINTER(CQuantConfig)])
_sig("qfb_quant_pass_host_submit", _i32, [_vp, _i32, ctypes.POINTER(CHostPoint), _i32,
                                          ctypes.POINTER(CQuantConfig), _i32])
_sig("qfb_quant_pass_host_wait", _i32, [_vp, _i32])
_sig("qfb_fake_quantize_backward_host", _i32, [_vp, _i32, _vp, _vp, _vp, _i64, _i64, _i64, _pd,
                                                ctypes.POINTER(CQuantConfig), _pd, _i32])


def lib() -> ctypes.CDLL:
    """The loaded libqfb.so handle (raw C-ABI)."""
    return _lib


def check(status: int) -> None:
    """Raise the qf exception mirroring a qfb_status."""
    if status != 0:
        msg = _lib.qfb_last_error().decode(errors="replace")
        raise _STATUS.get(status, QfError)(msg)


def build_info() -> str:
    return _lib.qfb_build_info().decode()

# ------------------------------------------------------------- config --


@dataclasses.dataclass
class QuantConfig:
    """qf::QuantConfig (quant.hpp:35-61)."""
    bits: int = 8
    s_min: float = 1e-6
    s_min_half: float = 1e-4
    s_max: float = 64.0
    eps: float = 1e-8

    def q_max(self) -> int:
        return (1 << (self.bits - 1)) - 1

    def s_min_for(self, precision: int) -> float:
        return self.s_min_half if precision == PREC_HALF else self.s_min

    def to_c(self) -> CQuantConfig:
        return CQuantConfig(self.bits, 0, self.s_min, self.s_min_half, self.s_max, self.eps)

    def validate(self) -> None:
        c = self.to_c()
        check(_lib.qfb_quant_config_validate(ctypes.byref(c)))


def _cfg(cfg: Optional[QuantConfig]) -> QuantConfig:
    return cfg if cfg is not None else QuantConfig()


def _darr(vals: Sequence[float]):
    arr = (ctypes.c_double * max(len(vals), 1))(*vals)
    return arr

# ------------------------------------------------------ host scale math --


def softplus(x: float) -> float:
    return _lib.qfb_softplus(float(x))


def sigmoid(x: float) -> float:
    return _lib.qfb_sigmoid(float(x))


def softplus_inv(y: float) -> float:
    out = ctypes.c_double()
    check(_lib.qfb_softplus_inv(float(y), ctypes.byref(out)))
    return out.value


def resolve_scale(log_s: Union[float, Sequence[float]], cfg: Optional[QuantConfig] = None,
                  precision: int = PREC_FULL):
    """quant.hpp:95-109. Scalar in -> float out; sequence in -> list out."""
    scalar = not isinstance(log_s, (list, tuple)) and not hasattr(log_s, "__len__")
    vals = [float(log_s)] if scalar else [float(v) for v in log_s]
    c = _cfg(cfg).to_c()
    out = _darr([0.0] * len(vals))
    check(_lib.qfb_resolve_scales(_darr(vals), len(vals), ctypes.byref(c), precision, out))
    res = [out[i] for i in range(len(vals))]
    return res[0] if scalar else res


def scale_grad_factors(log_s: Sequence[float], cfg: Optional[QuantConfig] = None,
                       precision: int = PREC_FULL):
    """(s, chain) per scale, quant.hpp:241-244 / 281-284."""
    vals = [float(v) for v in log_s]
    c = _cfg(cfg).to_c()
    s = _darr([0.0] * len(vals))
    ch = _darr([0.0] * len(vals))
    check(_lib.qfb_scale_grad_factors(_darr(vals), len(vals), ctypes.byref(c), precision, s, ch))
    return [s[i] for i in range(len(vals))], [ch[i] for i in range(len(vals))]


def cast_scales_f32(s: Sequence[float]):
    vals = [float(v) for v in s]
    out = (ctypes.c_float * max(len(vals), 1))()
    check(_lib.qfb_cast_scales_f32(_darr(vals), len(vals), out))
    return [out[i] for i in range(len(vals))]

# ------------------------------------------------------------- context --


class Context:
    """qfb_ctx: one per (device, stream). Externally single-threaded."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self.device = device
        h = _vp()
        check(_lib.qfb_ctx_create(device, _vp(stream or 0), ctypes.byref(h)))
        self.handle = h

    def set_stream(self, stream: Optional[int]) -> None:
        check(_lib.qfb_ctx_set_stream(self.handle, _vp(stream or 0)))

    def set_option(self, option: int, value: int) -> None:
        """qfb_ctx_set_option, e.g. (OPT_BWD_HALF_FP32, 1): float32 terms in
        the binary16 backward (d_input bitwise, d_log_s within tolerance)."""
        check(_lib.qfb_ctx_set_option(self.handle, option, value))

    def sync(self) -> None:
        check(_lib.qfb_ctx_sync(self.handle))

    def join(self) -> None:
        """qfb_ctx_join: the context stream waits for its side-stream work
        (QFB_OPT_BWD_ASYNC_FINISH's finisher)."""
        check(_lib.qfb_ctx_join(self.handle))

    @property
    def launch_count(self) -> int:
        return _lib.qfb_ctx_launch_count(self.handle)

    @property
    def sm_count(self) -> int:
        return _lib.qfb_ctx_sm_count(self.handle)

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.qfb_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


_CTX = {}


def default_context(device: Optional[int] = None) -> Context:
    """Per-device context bound to torch's current stream of that device."""
    import torch
    if device is None:
        device = torch.cuda.current_device()
    ctx = _CTX.get(device)
    if ctx is None:
        ctx = _CTX[device] = Context(device)
    ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)
    return ctx

# -------------------------------------------------- tensor-level ops --


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float16:
        return F16
    raise ValueError(f"unsupported dtype {t.dtype} (float32 / float16 only)")


def _layout(x, nscale: int, channel_axis: int):
    """[outer, channels, inner] view of x for a scale vector of nscale."""
    shape = list(x.shape)
    if nscale == 1 and channel_axis is None:
        return 1, 1, x.numel()
    ax = 0 if channel_axis is None else channel_axis
    if len(shape) == 0 or shape[ax] != nscale:
        raise ShapeError(f"fake_quantize: per-channel scale length {nscale} != dim {ax} of {shape}")
    outer = 1
    for d in shape[:ax]:
        outer *= d
    inner = 1
    for d in shape[ax + 1:]:
        inner *= d
    return outer, nscale, inner


def _scale_list(s) -> list:
    if isinstance(s, (list, tuple)):
        return [float(v) for v in s]
    if hasattr(s, "tolist") and not isinstance(s, float):
        v = s.tolist()
        return [float(a) for a in (v if isinstance(v, list) else [v])]
    return [float(s)]


def fake_quantize(x, s, cfg: Optional[QuantConfig] = None, precision: Optional[int] = None,
                  channel_axis: Optional[int] = None, out=None, ctx: Optional[Context] = None):
    """qf::fake_quantize (quant.hpp:136 per-tensor, :150 per-channel).

    ``s``: a positive float (per-tensor) or a sequence of positive floats
    (per-channel along ``channel_axis``, default axis 0 like the reference).
    float16 tensors are EmulatedHalf; ``precision=PREC_HALF`` on a float32
    tensor re-rounds the result onto the binary16 grid. A non-finite result
    on the half path raises NonFiniteError (tensor.hpp:160).
    """
    import torch
    cfg = _cfg(cfg)
    svals = _scale_list(s)
    per_channel = isinstance(s, (list, tuple)) or (hasattr(s, "__len__") and len(svals) != 1) \
        or channel_axis is not None
    sf = cast_scales_f32(svals)
    outer, ch, inner = _layout(x, len(svals), channel_axis if per_channel else None)
    if not x.is_cuda:
        raise ValueError("fake_quantize: tensor must live on a CUDA device")
    x = x.contiguous()
    y = torch.empty_like(x) if out is None else out
    ctx = ctx or default_context(x.device.index)
    ds = torch.tensor(sf, dtype=torch.float32, device=x.device)
    dt = _dtype_code(x)
    half = dt == F16 or precision == PREC_HALF
    flags = FLAG_HALF_GRID if (half and dt == F32) else 0
    check(_lib.qfb_fq_fwd(ctx.handle, dt, _vp(x.data_ptr()), _vp(y.data_ptr()), outer, ch, inner,
                          _vp(ds.data_ptr()), cfg.q_max(), flags))
    if half:
        ctx.sync()
    return y


def int8_codes(x, s, cfg: Optional[QuantConfig] = None, channel_axis: Optional[int] = None,
               ctx: Optional[Context] = None):
    """qf::int8_codes (quant.hpp:174-207)."""
    import torch
    cfg = _cfg(cfg)
    svals = _scale_list(s)
    per_channel = isinstance(s, (list, tuple)) or channel_axis is not None
    sf = cast_scales_f32(svals)
    outer, ch, inner = _layout(x, len(svals), channel_axis if per_channel else None)
    x = x.contiguous()
    codes = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    ctx = ctx or default_context(x.device.index)
    ds = torch.tensor(sf, dtype=torch.float32, device=x.device)
    check(_lib.qfb_int8_codes(ctx.handle, _dtype_code(x), _vp(x.data_ptr()), _vp(codes.data_ptr()),
                              outer, ch, inner, _vp(ds.data_ptr()), cfg.q_max()))
    return codes


@dataclasses.dataclass
class FakeQuantGrad:
    """qf::FakeQuantGrad (quant.hpp:209-212)."""
    d_input: object
    d_log_scale: list


def fake_quantize_backward(x, log_s, cfg: Optional[QuantConfig], upstream,
                           precision: int = PREC_FULL, channel_axis: Optional[int] = None,
                           need_d_input: bool = True, ctx: Optional[Context] = None):
    """qf::fake_quantize_backward (quant.hpp:233 per-tensor, :261 per-channel).

    Bit-identical to the reference: per-element terms in double and the
    fixed pairwise reduction tree. With channel_axis > 0 (outer > 1 rows per
    channel) the per-row results are accumulated in row order like the
    trainer's ``g += grad`` (frontend.hpp:222-228).
    """
    import torch
    cfg = _cfg(cfg)
    if tuple(x.shape) != tuple(upstream.shape):
        raise ShapeError(f"fake_quantize_backward: x {list(x.shape)} vs upstream {list(upstream.shape)}")
    lvals = _scale_list(log_s)
    per_channel = isinstance(log_s, (list, tuple)) or channel_axis is not None
    outer, ch, inner = _layout(x, len(lvals), channel_axis if per_channel else None)
    s64, chain = scale_grad_factors(lvals, cfg, precision)
    dev = x.device
    fac = torch.tensor(s64 + chain, dtype=torch.float64, device=dev)
    dls = torch.empty(ch, dtype=torch.float64, device=dev)  # accumulate = 0: every entry is written
    x = x.contiguous()
    upstream = upstream.contiguous()
    if upstream.dtype != x.dtype:
        raise ValueError("fake_quantize_backward: x and upstream must share a dtype")
    dx = torch.empty_like(x) if need_d_input else None
    ctx = ctx or default_context(dev.index)
    check(_lib.qfb_fq_bwd(ctx.handle, _dtype_code(x), _vp(x.data_ptr()), _vp(upstream.data_ptr()),
                          _vp(dx.data_ptr() if dx is not None else 0), outer, ch, inner,
                          _vp(fac.data_ptr()), _vp(fac.data_ptr() + 8 * ch), cfg.q_max(),
                          _vp(dls.data_ptr()), 0))
    return FakeQuantGrad(dx, dls.cpu().tolist())


def fq_chain(a, b=None, scales=(), act: int = ACT_RELU, half: bool = False, preact: bool = False,
             cfg: Optional[QuantConfig] = None, channel_axis: Optional[int] = None,
             ctx: Optional[Context] = None):
    """Fused maybe_half(act(a + b)) -> FQ x len(scales) (exec.hpp:438-451).

    ``scales``: up to two entries, each a float (per-tensor) or a sequence
    (per-channel along channel_axis). Returns (outputs, preact-or-None).
    """
    import torch
    cfg = _cfg(cfg)
    if len(scales) > 2:
        raise ValueError("fq_chain: at most 2 outputs")
    a = a.contiguous()
    if b is not None:
        if tuple(b.shape) != tuple(a.shape):
            raise ShapeError(f"add: shape mismatch {list(a.shape)} vs {list(b.shape)}")
        b = b.contiguous()
    nscale = len(_scale_list(scales[0])) if scales else 1
    per_channel = channel_axis is not None or (scales and isinstance(scales[0], (list, tuple)))
    outer, ch, inner = _layout(a, nscale, channel_axis if per_channel else None)
    ctx = ctx or default_context(a.device.index)
    d = CChainDesc()
    d.a = a.data_ptr()
    d.b = b.data_ptr() if b is not None else None
    pre = torch.empty_like(a) if preact else None
    d.preact = pre.data_ptr() if pre is not None else None
    outs, keep = [], []
    for k, s in enumerate(scales):
        sv = cast_scales_f32(_scale_list(s))
        if len(sv) != ch:
            raise ShapeError("fq_chain: scale vectors must have the same length")
        ds = torch.tensor(sv, dtype=torch.float32, device=a.device)
        keep.append(ds)
        y = torch.empty_like(a)
        outs.append(y)
        d.y[k] = y.data_ptr()
        d.scale[k] = ds.data_ptr()
    d.outer, d.channels, d.inner = outer, ch, inner
    d.n_out = len(scales)
    d.act = act
    d.dtype = _dtype_code(a)
    d.q_max = cfg.q_max()
    d.flags = FLAG_HALF_GRID if (half and d.dtype == F32) else 0
    check(_lib.qfb_fq_chain(ctx.handle, ctypes.byref(d)))
    if half or d.dtype == F16:
        ctx.sync()
    return outs, pre


def fill_rng(t, seed: int, stream: int, kind: int = 1, lo: float = 1.0, hi: float = 0.0,
             offset: int = 0, ctx: Optional[Context] = None):
    """Counter-RNG synthetic data on the device (rng.hpp:24-50)."""
    ctx = ctx or default_context(t.device.index)
    check(_lib.qfb_fill_rng(ctx.handle, _dtype_code(t), _vp(t.data_ptr()), t.numel(), seed, stream,
                            offset, kind, lo, hi))
    return t


# ------------------------------------------------------ execution plan --

MODE_PER_OPERATOR, MODE_FUSED = 0, 1
POLICY_FULL_ONLY, POLICY_HALF_ACTIVATIONS = 0, 1


@dataclasses.dataclass
class ExecutionPlan:
    """qf::ExecutionPlan (exec.hpp:55-65); `threads` has no GPU meaning."""
    mode: int = MODE_FUSED
    policy: int = POLICY_FULL_ONLY
    fallback_enabled: bool = True
    cache_weights: bool = False
    fault_inject_layer: int = -1

    def to_c(self) -> CExecPlan:
        return CExecPlan(self.mode, self.policy, int(self.fallback_enabled), int(self.cache_weights),
                         self.fault_inject_layer, 0)


class ExecutionContext:
    """The quantization part of qf::ExecutionContext + run_quant_conv
    (exec.hpp:182-405) on the GPU: `quant_layer` returns (qa, qw) for the
    caller's convolution; `trace` holds the modeled counters."""

    def __init__(self, plan: ExecutionPlan, ctx: Optional[Context] = None, device: int = 0):
        self.plan = plan
        self.ctx = ctx or default_context(device)
        h = _vp()
        c = plan.to_c()
        check(_lib.qfb_exec_create(self.ctx.handle, ctypes.byref(c), ctypes.byref(h)))
        self.handle = h

    def quant_layer(self, index: int, x, weight, log_w: Sequence[float], log_a: float,
                    cfg: Optional[QuantConfig] = None):
        import torch
        cfg = _cfg(cfg)
        w = weight.contiguous().float()
        c_out = w.shape[0]
        per = w.numel() // c_out
        lw = (ctypes.c_double * c_out)(*[float(v) for v in log_w])
        L = CQuantLayer(index, 0, w.data_ptr(), c_out, per, ctypes.cast(lw, _vp), float(log_a))
        x = x.contiguous()
        qa = torch.empty_like(x)
        qw_buf = None if self.plan.cache_weights else torch.empty_like(w)
        out = _vp()
        cc = cfg.to_c()
        check(_lib.qfb_exec_quant_layer(self.handle, ctypes.byref(L), ctypes.byref(cc), _dtype_code(x),
                                        _vp(x.data_ptr()), x.numel(), _vp(qa.data_ptr()),
                                        _vp(qw_buf.data_ptr() if qw_buf is not None else 0),
                                        ctypes.byref(out)))
        self.ctx.sync()
        if qw_buf is not None and out.value == qw_buf.data_ptr():
            return qa, qw_buf
        # plan-owned cache buffer: return a copy (the cache stays private)
        return qa, _device_view(out.value, w.numel() * 4, w.device).view(torch.float32).view_as(w).clone()

    @property
    def trace(self) -> CExecTrace:
        t = CExecTrace()
        check(_lib.qfb_exec_trace_get(self.handle, ctypes.byref(t)))
        return t

    def close(self):
        if getattr(self, "handle", None):
            _lib.qfb_exec_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _device_view(ptr: int, nbytes: int, device):
    """uint8 torch view of a library-owned device buffer."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 2}
    return torch.as_tensor(_View(), device=device)


def model_layer_counts(plan: ExecutionPlan, n_act: int, c_out: int, per: int, weights_cached: bool = False,
                       fused_fails: bool = False) -> CExecTrace:
    """Host-only modeled counter increments of one layer (exec.hpp:199-216)."""
    t = CExecTrace()
    c = plan.to_c()
    check(_lib.qfb_exec_model_layer(ctypes.byref(c), n_act, c_out, per, int(weights_cached),
                                    int(fused_fails), ctypes.byref(t)))
    return t


# ------------------------------------------------- QAT step --

_sig("qfb_distill_pair", _i32, [_vp, _vp, _vp, _i64, _i64, ctypes.c_double, ctypes.c_double, _vp, _vp])
_sig("qfb_distill_batch", _i32, [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_double, ctypes.c_double, _vp, _vp])
_sig("qfb_fold_rows", _i32, [_vp, _vp, _i64, _i64, _vp, _vp])
_sig("qfb_adam_bias_corrections", _i32, [ctypes.c_double, ctypes.c_double, _i64,
                                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)])
_sig("qfb_adam_step", _i32, [_vp, _vp, _vp, _vp, _vp, _i64, ctypes.c_double, ctypes.c_double,
                             ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, _vp])


def distill_pair(student, teacher, lambda_cos: float, grad_scale: float = 1.0,
                 ctx: Optional[Context] = None):
    """One tensor pair of qf::distill_loss (distill.hpp:66-124) on the GPU:
    student/teacher float32 CUDA tensors [C, ...]. Returns (d_student,
    out2) with out2 a float64 CUDA tensor {mse, mean cosine}; d_student is
    scaled float(d * grad_scale) like the trainer's 1/chunk_len scaling."""
    import torch
    if tuple(student.shape) != tuple(teacher.shape):
        raise ShapeError(f"distill_loss: student {list(student.shape)} vs teacher {list(teacher.shape)}")
    if student.dim() < 1 or student.shape[0] < 1:
        raise ShapeError("distill_loss: channel dim must be >= 1")
    if student.dtype != torch.float32 or teacher.dtype != torch.float32:
        raise ValueError("distill_loss: float32 tensors expected (promote_full first)")
    s = student.contiguous()
    t = teacher.contiguous()
    c = s.shape[0]
    hw = s.numel() // c
    d = torch.empty_like(s)
    out2 = torch.empty(2, dtype=torch.float64, device=s.device)
    ctx = ctx or default_context(s.device.index)
    check(_lib.qfb_distill_pair(ctx.handle, _vp(s.data_ptr()), _vp(t.data_ptr()), c, hw, lambda_cos,
                                grad_scale, _vp(d.data_ptr()), _vp(out2.data_ptr())))
    return d, out2


def distill_loss(f_s, f_t, i_s, i_t, lambda_cos: float, grad_scale: float = 1.0,
                 ctx: Optional[Context] = None):
    """qf::distill_loss (distill.hpp:126-141): returns (dict of total, mse_f,
    mse_i, cos_f, cos_i as Python floats, d_features, d_descriptors)."""
    df, f2 = distill_pair(f_s, f_t, lambda_cos, grad_scale, ctx)
    di, i2 = distill_pair(i_s, i_t, lambda_cos, grad_scale, ctx)
    mf, cf = f2.tolist()
    mi, ci = i2.tolist()
    total = mf + mi + lambda_cos * (1.0 - cf) + lambda_cos * (1.0 - ci)
    return {"total": total, "mse_f": mf, "mse_i": mi, "cos_f": cf, "cos_i": ci}, df, di


def adam_bias_corrections(beta1: float, beta2: float, t: int):
    b1, b2 = ctypes.c_double(), ctypes.c_double()
    check(_lib.qfb_adam_bias_corrections(beta1, beta2, t, ctypes.byref(b1), ctypes.byref(b2)))
    return b1.value, b2.value


_sig("qfb_adam_bias_table", _i32, [ctypes.c_double, ctypes.c_double, _i64, _vp])
_sig("qfb_adam_step_dev", _i32, [_vp, _vp, _vp, _vp, _vp, _i64, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, _vp, _i64, _vp, _vp, _i64, _vp])


class DeviceAdam:
    """Adam over a flattened float64 CUDA scale vector whose step counter
    lives on the device (qfb_adam_step_dev), so a captured CUDA graph
    replays true successive steps: t = non-skipped steps + 1
    (distill.hpp:262-264), bias corrections from a host-pow table."""

    def __init__(self, params, beta1: float = 0.9, beta2: float = 0.999, lr: float = 5e-3,
                 eps: float = 1e-8, t_max: int = 4096):
        import numpy as np
        import torch
        dev = params.device
        self.params, self.b1, self.b2, self.lr, self.eps, self.t_max = params, beta1, beta2, lr, eps, t_max
        self.m = torch.zeros_like(params)
        self.v = torch.zeros_like(params)
        tab = np.empty(2 * t_max, dtype=np.float64)
        check(_lib.qfb_adam_bias_table(beta1, beta2, t_max, tab.ctypes.data))
        self.table = torch.from_numpy(tab).to(dev)
        self.counters = torch.zeros(3, dtype=torch.int64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)

    def step(self, grads, loss=None, ctx: Optional[Context] = None) -> None:
        ctx = ctx or default_context(self.params.device.index)
        nl = 0 if loss is None else loss.numel()
        check(_lib.qfb_adam_step_dev(ctx.handle, _vp(self.params.data_ptr()), _vp(self.m.data_ptr()),
                                     _vp(self.v.data_ptr()), _vp(grads.data_ptr()), self.params.numel(),
                                     self.b1, self.b2, self.lr, self.eps, _vp(self.table.data_ptr()),
                                     self.t_max, _vp(self.counters.data_ptr()),
                                     _vp(loss.data_ptr() if loss is not None else None), nl,
                                     _vp(self.flag.data_ptr())))


def adam_step(params, m, v, grads, t: int, lr: float, beta1: float = 0.9, beta2: float = 0.999,
              eps: float = 1e-8, skipped=None, ctx: Optional[Context] = None):
    """Adam over the flattened scale vector (distill.hpp:264-279), in place
    on float64 CUDA tensors; the update is skipped when any gradient is
    non-finite. Returns the device u32 counter of non-finite gradients."""
    import torch
    bc1, bc2 = adam_bias_corrections(beta1, beta2, t)
    if skipped is None:
        skipped = torch.zeros(1, dtype=torch.int32, device=params.device)
    ctx = ctx or default_context(params.device.index)
    check(_lib.qfb_adam_step(ctx.handle, _vp(params.data_ptr()), _vp(m.data_ptr()), _vp(v.data_ptr()),
                             _vp(grads.data_ptr()), params.numel(), beta1, beta2, lr, eps, bc1, bc2,
                             _vp(skipped.data_ptr())))
    return skipped


def fold_rows_device(rows, into=None, ctx: Optional[Context] = None):
    """((into + r0) + r1) + ... over the rows of a [R, n] float64 CUDA tensor
    in one launch (qfb_fold_rows)."""
    import torch
    rows = rows.contiguous()
    out = torch.empty(rows.shape[1:], dtype=torch.float64, device=rows.device)
    ctx = ctx or default_context(rows.device.index)
    check(_lib.qfb_fold_rows(ctx.handle, _vp(rows.data_ptr()), rows.shape[0], out.numel(),
                             _vp(into.contiguous().data_ptr() if into is not None else None), _vp(out.data_ptr())))
    return out


# ---- multi-GPU exchange through the C-ABI (qfb_nccl.cpp) -------------------
_sig("qfb_nccl_available", _i32, [])
_sig("qfb_nccl_comm_init_all", _i32, [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_vp)])
_sig("qfb_nccl_get_unique_id", _i32, [_vp])
_sig("qfb_nccl_comm_init_rank", _i32, [ctypes.POINTER(_vp), ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int])
NCCL_UNIQUE_ID_BYTES = 128


def nccl_unique_id() -> bytes:
    """qfb_nccl_get_unique_id: the 128-byte id rank 0 broadcasts."""
    buf = ctypes.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    check(_lib.qfb_nccl_get_unique_id(buf))
    return buf.raw


class NcclRankComm:
    """One rank's communicator of a one-process-per-GPU job
    (qfb_nccl_comm_init_rank). `uid` comes from nccl_unique_id() on rank 0,
    broadcast by the launcher's plumbing."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        if len(uid) != NCCL_UNIQUE_ID_BYTES:
            raise ValueError("nccl unique id must be 128 bytes")
        self.nranks, self.rank, self.device = nranks, rank, device
        h = _vp()
        buf = ctypes.create_string_buffer(uid, NCCL_UNIQUE_ID_BYTES)
        check(_lib.qfb_nccl_comm_init_rank(ctypes.byref(h), nranks, buf, rank, device))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            _lib.qfb_nccl_comm_destroy(self.handle)
            self.handle = None
_sig("qfb_nccl_comm_destroy", _i32, [_vp])
_sig("qfb_allreduce_scale_grads", _i32, [_vp, _vp, _vp, _i64])
_sig("qfb_gather_fold_scale_grads", _i32, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp])


def nccl_available() -> bool:
    """True when libqfb found an NCCL library to dlopen."""
    return _lib.qfb_nccl_available() == 0


class NcclComms:
    """Single-process communicators, one per device (ncclCommInitAll), for
    the C-ABI exchange: the process model of SURVEY §8e. With torchrun
    (one process per GPU) use dist.gather_fold instead."""

    def __init__(self, devices):
        self.devices = list(devices)
        n = len(self.devices)
        arr = (ctypes.c_int * n)(*self.devices)
        self._comms = (_vp * n)()
        check(_lib.qfb_nccl_comm_init_all(n, arr, self._comms))

    def __getitem__(self, i):
        return self._comms[i]

    def close(self):
        for i in range(len(self.devices)):
            if self._comms[i]:
                _lib.qfb_nccl_comm_destroy(self._comms[i])
                self._comms[i] = None


def gather_fold_scale_grads(comm, rows, nranks: int, into=None, ctx: Optional[Context] = None):
    """qfb_gather_fold_scale_grads: all-gather this rank's gradient rows
    [R, n] (float64 CUDA) over `comm` (nranks ranks) and fold all ranks'
    rows in rank-major (= frame) order; returns the folded [n] vector."""
    import torch
    rows = rows.contiguous()
    ctx = ctx or default_context(rows.device.index)
    R, n = rows.shape[0], rows[0].numel()
    gathered = torch.empty((R * nranks, n), dtype=torch.float64, device=rows.device)
    out = torch.empty(n, dtype=torch.float64, device=rows.device)
    check(_lib.qfb_gather_fold_scale_grads(ctx.handle, _vp(comm), _vp(rows.data_ptr()), R, n,
                                           _vp(gathered.data_ptr()),
                                           _vp(into.contiguous().data_ptr() if into is not None else None),
                                           _vp(out.data_ptr())))
    return out


def allreduce_scale_grads(comm, grads, ctx: Optional[Context] = None):
    """qfb_allreduce_scale_grads: in-place ncclAllReduce(sum) of a float64
    CUDA vector (bits depend on the GPU count; see gather_fold)."""
    ctx = ctx or default_context(grads.device.index)
    check(_lib.qfb_allreduce_scale_grads(ctx.handle, _vp(comm), _vp(grads.data_ptr()), grads.numel()))
    return grads
