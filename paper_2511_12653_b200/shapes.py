"""DPVO front-end quant-point catalogue and algorithmic byte model (pure Python).

No native code: importing this module (or the package for it) maps no
shared library, so the reference CPU arm of bench.py can build the same
workload without loading libqfb.so.

Shapes: the reference ships only a 10-layer toy roster
(model.hpp:134-143); the DPVO encoder shapes are the public BasicEncoder4's
(22 convs, quant point = conv input). Multi-consumer points read
their tensor once and write one output per consumer (exec.hpp:440-451):
the image feeds both encoders' conv1; each layer2.0 input feeds conv1 and
downsample.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

H, W = 480, 640
# activation codes of qfb_chain_desc.act (include/qfb.h)
ACT_NONE, ACT_RELU, ACT_GELU = 0, 1, 2


@dataclass
class QuantPoint:
    name: str
    channels: int
    height: int
    width: int
    consumers: List[str] = field(default_factory=list)

    @property
    def inner(self) -> int:
        return self.height * self.width

    @property
    def numel(self) -> int:
        return self.channels * self.inner


def dpvo_quant_points(h: int = H, w: int = W) -> List[QuantPoint]:
    """The 19 activation tensors / 22 quant points of one frame."""
    pts = [QuantPoint("image", 3, h, w, ["fnet.conv1", "inet.conv1"])]
    h2, w2, h4, w4 = h // 2, w // 2, h // 4, w // 4
    for enc in ("fnet", "inet"):
        for blk in ("layer1.0", "layer1.1"):
            for cv in ("conv1", "conv2"):
                pts.append(QuantPoint(f"{enc}.{blk}.{cv}.in", 32, h2, w2, [f"{enc}.{blk}.{cv}"]))
        pts.append(QuantPoint(f"{enc}.layer2.0.in", 32, h2, w2,
                              [f"{enc}.layer2.0.conv1", f"{enc}.layer2.0.downsample"]))
        pts.append(QuantPoint(f"{enc}.layer2.0.conv2.in", 64, h4, w4, [f"{enc}.layer2.0.conv2"]))
        for cv in ("conv1", "conv2"):
            pts.append(QuantPoint(f"{enc}.layer2.1.{cv}.in", 64, h4, w4, [f"{enc}.layer2.1.{cv}"]))
        pts.append(QuantPoint(f"{enc}.conv2.in", 64, h4, w4, [f"{enc}.conv2"]))
    return pts


def frame_bytes(points: List[QuantPoint], esize: int) -> dict:
    """Algorithmic HBM bytes per frame: forward reads each
    tensor once and writes one output per consumer; backward reads x and
    upstream and writes d_input per consumer."""
    uniq = sum(p.numel for p in points)
    qp = sum(p.numel * len(p.consumers) for p in points)
    return {"fwd": (uniq + qp) * esize, "bwd": 3 * qp * esize, "unique_elems": uniq,
            "quant_point_elems": qp, "fwd_int8": uniq * esize + qp}


# ------------------------------------------------------------------------
# BASELINE config 3: fused quant -> act -> quant chains over a sliding
# window (exec.hpp:431-451 residual joins maybe_half(relu(add(a, b))) and
# multi-consumer points).
# ------------------------------------------------------------------------

@dataclass
class ChainPoint:
    name: str
    outer: int
    channels: int
    inner: int
    consumers: int     # K fake-quant outputs from one read
    act: int           # ACT_NONE / ACT_RELU / ACT_GELU (GELU variant)
    residual: bool     # a + b join before the activation

    @property
    def numel(self) -> int:
        return self.outer * self.channels * self.inner


# Encoder points whose input is a residual join relu(x + y) (BasicEncoder4:
# the outputs of layer1.0, layer1.1, layer2.0, layer2.1).
_RESIDUAL = ("layer1.1.conv1.in", "layer2.0.in", "layer2.1.conv1.in", "conv2.in")


def window_chain_points(frames: int = 15, patches: int = 96, gelu: bool = False,
                        h: int = H, w: int = W) -> List[ChainPoint]:
    """Every activation quant point of a `frames`-frame window: the 19
    per-frame encoder tensors (outer = frames, per-channel scales) and the
    patch / update-operator inputs of the window (gmap, imap, and
    per-edge corr / net / inp for E = patches * frames * frames edges,
    per-tensor scales)."""
    act = ACT_GELU if gelu else ACT_RELU
    pts = []
    for p in dpvo_quant_points(h, w):
        first = p.name == "image"
        res = any(p.name.endswith(r) for r in _RESIDUAL)
        pts.append(ChainPoint(p.name, frames, p.channels, p.inner, len(p.consumers),
                              ACT_NONE if first else act, res))
    n_patch = patches * frames
    edges = patches * frames * frames
    # per-tensor scales: one [1, 1, n] row (same arithmetic, 16-byte units)
    pts += [ChainPoint("patch.gmap", 1, 1, n_patch * 128 * 9, 1, ACT_NONE, False),
            ChainPoint("patch.imap", 1, 1, n_patch * 384, 1, ACT_NONE, False),
            ChainPoint("update.corr", 1, 1, edges * 2 * 49 * 9, 1, ACT_NONE, False),
            ChainPoint("update.net", 1, 1, edges * 384, 1, act, True),
            ChainPoint("update.inp", 1, 1, edges * 384, 1, act, False)]
    return pts
