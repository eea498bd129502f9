"""paper_2511_12653_b200 — B200-native fused fake-quantization (qfb).

Python mirror of the reference operator API (quantfuse, namespace ``qf``,
/root/reference/proj/include/quantfuse/quant.hpp) on top of the C-ABI in
``include/qfb.h``. Every call goes through ``libqfb.so`` (hand-written
sm_100a kernels). There is no CPU or eager-PyTorch fallback: if the library
is missing, the first use of the package raises ImportError.

PyTorch is used only as plumbing: device memory (``torch.Tensor`` on
``cuda``) and the current CUDA stream.

Reference names kept: ``QuantConfig``, ``resolve_scale``, ``softplus``,
``sigmoid``, ``softplus_inv``, ``fake_quantize``, ``int8_codes``,
``fake_quantize_backward`` (returning ``FakeQuantGrad``), and the error
taxonomy ``ShapeError``/``ValueError``/``IoError``/``NonFiniteError``/
``FusedPathError`` (errors.hpp:11-33, exec.hpp:51).

The binding lives in ``_api`` and is loaded LAZILY, on the first access of
any package attribute (``paper_2511_12653_b200.fake_quantize``, ``from
paper_2511_12653_b200 import Context``, ...). Pure-Python submodules
(``shapes``: the DPVO quant-point catalogue and byte model) import without
mapping libqfb.so, so the reference CPU arm of bench.py runs with no native
code of this package in its process.
"""
from __future__ import annotations

import importlib as _importlib

_API = None


def _load():
    global _API
    if _API is None:
        _API = _importlib.import_module("._api", __name__)
    return _API


def __getattr__(name):
    if name.startswith("__"):
        raise AttributeError(name)
    try:
        return getattr(_load(), name)
    except AttributeError:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}") from None


def __dir__():
    return sorted(set(globals()) | set(dir(_load())))
