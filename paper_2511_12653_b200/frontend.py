"""DPVO front-end quant pass: every activation quant point of the two
BasicEncoder4 encoders (fnet, inet) for a batch of 480x640 frames, run as ONE
fused forward launch and ONE backward launch through the C-ABI tables.

This is the B200 counterpart of the quant portion of the reference's
front-end walk (exec.hpp:416-460 run_frontend / frontend.hpp:170-258
forward_train + backward_train): per quant point the activation fake-quant
forward (exec.hpp:353-361) and the scale-only backward
(frontend.hpp:226-229 -> quant.hpp:261-294). The convolutions themselves are
out of scope (cuDNN territory).

Shapes: the reference ships only a 10-layer toy roster
(model.hpp:134-143); the DPVO encoder shapes are the public BasicEncoder4's
(22 convs, quant point = conv input). Multi-consumer points read
their tensor once and write one output per consumer (exec.hpp:440-451):
the image feeds both encoders' conv1; each layer2.0 input feeds conv1 and
downsample.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import (ACT_GELU, ACT_NONE, ACT_RELU, CBwdDesc, CChainDesc, CFqDesc, F16, F32, Context, check,
               lib, scale_grad_factors)

H, W = 480, 640


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


class FrontendQuantPass:
    """Device buffers + C-ABI descriptor tables for `frames` frames of the
    DPVO activation set, per-channel scales (log-uniform [1e-3, 0.1],
    SURVEY §8d C2). `sets` independent input sets rotate so consecutive
    steps never hit L2-resident inputs."""

    def __init__(self, ctx: Context, frames: int = 1, dtype: str = "f32", sets: int = 1,
                 seed: int = 1, device=None, h: int = H, w: int = W, int8_out: bool = False,
                 grads_out=None):
        """int8_out: the forward emits the int8 codes of every quant point
        (QFB_FLAG_INT8_OUT, 1 byte per element) instead of the
        fake-quant values; the backward is unchanged."""
        import torch
        self.ctx = ctx
        self.frames = frames
        self.int8_out = int8_out
        self.dtype_code = F32 if dtype == "f32" else F16
        tdt = torch.float32 if dtype == "f32" else torch.float16
        self.esize = 4 if dtype == "f32" else 2
        dev = device if device is not None else torch.device("cuda", ctx.device)
        self.points = dpvo_quant_points(h, w)
        self.consumers = [(p, c) for p in self.points for c in p.consumers]
        rng = np.random.default_rng(seed)
        L = lib()
        # scales: per consumer, per channel
        self.log_s, self.s32, self.fac, self.dls = [], [], [], []
        n_grad = sum(p.channels for p, _ in self.consumers)
        self.dls_flat = (grads_out if grads_out is not None
                         else torch.zeros(n_grad, dtype=torch.float64, device=dev))
        assert self.dls_flat.numel() == n_grad and self.dls_flat.dtype == torch.float64
        goff = 0
        for p, _ in self.consumers:
            s = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), p.channels))
            ls = np.log(np.expm1(s))
            s64, chain = scale_grad_factors(ls.tolist())
            self.log_s.append(ls)
            self.s32.append(torch.tensor(np.array(s64, dtype=np.float64).astype(np.float32), device=dev))
            self.fac.append(torch.tensor(s64 + chain, dtype=torch.float64, device=dev))
            self.dls.append(self.dls_flat[goff:goff + p.channels])
            goff += p.channels
        # outputs shared across sets (written every step)
        ydt = torch.int8 if int8_out else tdt
        self.y = [torch.empty((frames, p.channels, p.height, p.width), dtype=ydt, device=dev)
                  for p, _ in self.consumers]
        self.dx = [torch.empty((frames, p.channels, p.height, p.width), dtype=tdt, device=dev)
                   for p, _ in self.consumers]
        self.sets = []
        for si in range(sets):
            xs = []
            for pi, p in enumerate(self.points):
                t = torch.empty((frames, p.channels, p.height, p.width), dtype=tdt, device=dev)
                check(L.qfb_fill_rng(ctx.handle, self.dtype_code, t.data_ptr(), t.numel(),
                                     seed + 1000 * si, pi, 0, 1, 1.0, 0.0))
                xs.append(t)
            ups = []
            for ci, (p, _) in enumerate(self.consumers):
                t = torch.empty((frames, p.channels, p.height, p.width), dtype=tdt, device=dev)
                check(L.qfb_fill_rng(ctx.handle, self.dtype_code, t.data_ptr(), t.numel(),
                                     seed + 1000 * si + 500, ci, 0, 1, 1.0, 0.0))
                ups.append(t)
            self.sets.append(self._tables(xs, ups))
        ctx.sync()

    def _tables(self, xs, ups):
        fwd, bwd = [], []
        ci = 0
        for pi, p in enumerate(self.points):
            d = CFqDesc()
            d.x = xs[pi].data_ptr()
            d.outer, d.channels, d.inner = self.frames, p.channels, p.inner
            d.n_out, d.q_max, d.flags = len(p.consumers), 127, (0x4 if self.int8_out else 0)
            for k in range(len(p.consumers)):
                d.y[k] = self.y[ci + k].data_ptr()
                d.scale[k] = self.s32[ci + k].data_ptr()
            fwd.append(d)
            for k in range(len(p.consumers)):
                b = CBwdDesc()
                b.x, b.up, b.dx = xs[pi].data_ptr(), ups[ci + k].data_ptr(), self.dx[ci + k].data_ptr()
                b.scale64 = self.fac[ci + k].data_ptr()
                b.chain = self.fac[ci + k].data_ptr() + 8 * p.channels
                b.d_log_s = self.dls[ci + k].data_ptr()
                b.outer, b.channels, b.inner = self.frames, p.channels, p.inner
                b.q_max, b.accumulate = 127, 0
                bwd.append(b)
            ci += len(p.consumers)
        ft = (CFqDesc * len(fwd))(*fwd)
        bt = (CBwdDesc * len(bwd))(*bwd)
        return {"x": xs, "up": ups, "fwd": ft, "nf": len(fwd), "bwd": bt, "nb": len(bwd)}

    def forward(self, set_index: int = 0, ctx: Context = None) -> None:
        """All quant points' forward of one input set, on `ctx`'s stream
        (default: the pass's context)."""
        s = self.sets[set_index]
        check(lib().qfb_fq_fwd_multi((ctx or self.ctx).handle, self.dtype_code, s["fwd"], s["nf"]))

    def backward(self, set_index: int = 0, ctx: Context = None) -> None:
        """All quant points' backward (+ finisher) of one input set. A second
        context (own stream and scratch) lets the backward of frame k run
        beside the forward of frame k+1."""
        s = self.sets[set_index]
        check(lib().qfb_fq_bwd_multi((ctx or self.ctx).handle, self.dtype_code, s["bwd"], s["nb"]))

    def scale_grads(self):
        return self.dls_flat

    def bytes_per_step(self) -> dict:
        b = frame_bytes(self.points, self.esize)
        return {k: v * self.frames for k, v in b.items()}


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


class WindowChainPass:
    """Device buffers + one qfb_fq_chain_multi table for a window of chain
    points: per point a (the producing op's output), b (the skip tensor of a
    residual join), K fake-quant outputs."""

    def __init__(self, ctx: Context, frames: int = 15, patches: int = 96, gelu: bool = False,
                 dtype: str = "f32", seed: int = 3, device=None, h: int = H, w: int = W):
        import torch
        self.ctx = ctx
        self.points = window_chain_points(frames, patches, gelu, h, w)
        self.frames = frames
        self.dtype_code = F32 if dtype == "f32" else F16
        tdt = torch.float32 if dtype == "f32" else torch.float16
        self.esize = 4 if dtype == "f32" else 2
        dev = device if device is not None else torch.device("cuda", ctx.device)
        rng = np.random.default_rng(seed)
        L = lib()
        self.keep = []
        self.buffers = []   # per point: (a, b or None, [y], [scale]) for checks
        descs = []
        for pi, p in enumerate(self.points):
            a = torch.empty(p.numel, dtype=tdt, device=dev)
            check(L.qfb_fill_rng(ctx.handle, self.dtype_code, a.data_ptr(), a.numel(), seed, 2 * pi, 0,
                                 1, 1.0, 0.0))
            b = None
            if p.residual:
                b = torch.empty(p.numel, dtype=tdt, device=dev)
                check(L.qfb_fill_rng(ctx.handle, self.dtype_code, b.data_ptr(), b.numel(), seed,
                                     2 * pi + 1, 0, 1, 1.0, 0.0))
            d = CChainDesc()
            d.a = a.data_ptr()
            d.b = b.data_ptr() if b is not None else 0
            d.preact = 0
            d.outer, d.channels, d.inner = p.outer, p.channels, p.inner
            d.n_out, d.act, d.dtype, d.q_max, d.flags = p.consumers, p.act, self.dtype_code, 127, 0
            ys, ss = [], []
            for k in range(p.consumers):
                s = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), p.channels)).astype(np.float32)
                st = torch.from_numpy(s).to(dev)
                y = torch.empty(p.numel, dtype=tdt, device=dev)
                d.y[k], d.scale[k] = y.data_ptr(), st.data_ptr()
                self.keep += [st, y]
                ys.append(y)
                ss.append(s)
            self.buffers.append((a, b, ys, ss))
            self.keep += [a] + ([b] if b is not None else [])
            descs.append(d)
        self.table = (CChainDesc * len(descs))(*descs)
        self.n = len(descs)
        ctx.sync()

    def run(self) -> None:
        check(lib().qfb_fq_chain_multi(self.ctx.handle, self.table, self.n))

    def bytes_per_run(self) -> int:
        """Algorithmic bytes: read a (+ b), write K outputs."""
        return sum(p.numel * (1 + (1 if p.residual else 0) + p.consumers) * self.esize
                   for p in self.points)


# ------------------------------------------------------------------------
# BASELINE config 4: the scale-only QAT step of a batch of frames
# (distill.hpp:227-279) minus the convolutions (cuDNN territory): the fused
# fake-quant forward of every activation quant point, the distillation loss
# of every frame's fnet/inet outputs, the scale-only backward of every quant
# point (frame rows accumulate in frame order, the trainer's g += grad), and
# Adam on the scale vector. Features and upstream gradients are synthetic.
# ------------------------------------------------------------------------

class QatStep:
    """One scale-only QAT step over `frames` frames on one GPU (or this
    rank's shard); every piece is a qfb launch, capturable as one graph."""

    def __init__(self, ctx: Context, frames: int = 64, dtype: str = "f32", seed: int = 21, device=None,
                 h: int = H, w: int = W, lambda_cos: float = 1.0, lr: float = 5e-3,
                 n_weight_scales: int = 592):
        import torch
        from . import adam_bias_corrections
        self.ctx = ctx
        self.frames = frames
        self.lam = lambda_cos
        self.lr = lr
        dev = device if device is not None else torch.device("cuda", ctx.device)
        n_act = sum(p.channels * len(p.consumers) for p in dpvo_quant_points(h, w))
        self.n_act = n_act
        self.n_params = n_act + n_weight_scales
        # the backward writes its scale gradients straight into the optimizer's vector
        self.grads = torch.zeros(self.n_params, dtype=torch.float64, device=dev)
        self.fp = FrontendQuantPass(ctx, frames=frames, dtype=dtype, sets=1, seed=seed, device=dev, h=h, w=w,
                                    grads_out=self.grads[:n_act])
        h4, w4 = h // 4, w // 4
        L = lib()
        # synthetic student / teacher encoder outputs per frame (fnet 128, inet 384 channels)
        self.feat = []
        for k, c in enumerate((128, 384)):
            t = [torch.empty((frames, c, h4, w4), dtype=torch.float32, device=dev) for _ in range(2)]
            for j, tt in enumerate(t):
                check(L.qfb_fill_rng(ctx.handle, F32, tt.data_ptr(), tt.numel(), seed + 17, 10 * k + j, 0, 1,
                                     1.0, 0.0))
            self.feat.append((c, t[0], t[1], torch.empty_like(t[0])))
        # per pair (fnet, inet): [frames][mse, cos]; self.loss[f, k] views them
        self.loss_k = [torch.zeros((frames, 2), dtype=torch.float64, device=dev) for _ in range(2)]
        self.loss = torch.stack(self.loss_k, dim=1)  # refreshed by losses()
        # flattened trainable scales: the activation scales of the pass + weight scales
        self.params = torch.empty(self.n_params, dtype=torch.float64, device=dev)
        self.params[:n_act] = torch.from_numpy(np.concatenate(self.fp.log_s)).to(dev)
        self.params[n_act:] = -4.0
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.skipped = torch.zeros(1, dtype=torch.int32, device=dev)
        self.t = 1
        self.bc = adam_bias_corrections(0.9, 0.999, self.t)
        ctx.sync()
        torch.cuda.synchronize(dev)

    def run(self) -> None:
        """fwd (1 launch) -> per-frame distill loss (2 pairs) -> bwd (1
        launch + finisher, gradients land in the optimizer vector) -> Adam
        (2 launches). All on the context's stream."""
        from . import _lib, _vp
        self.fp.forward(0)
        inv = 1.0 / self.frames
        for k, (c, s, t, d) in enumerate(self.feat):
            # every frame's pair_loss in one batched call (per-frame trees)
            hw = s.shape[2] * s.shape[3]
            check(_lib.qfb_distill_batch(self.ctx.handle, _vp(s.data_ptr()), _vp(t.data_ptr()), self.frames, c,
                                         hw, self.lam, inv, _vp(d.data_ptr()), _vp(self.loss_k[k].data_ptr())))
        self.fp.backward(0)
        b1, b2 = self.bc
        check(_lib.qfb_adam_step(self.ctx.handle, _vp(self.params.data_ptr()), _vp(self.m.data_ptr()),
                                 _vp(self.v.data_ptr()), _vp(self.grads.data_ptr()), self.n_params, 0.9, 0.999,
                                 self.lr, 1e-8, b1, b2, _vp(self.skipped.data_ptr())))

    def losses(self):
        """[frames, 2 pairs, (mse, cos)] of the last run."""
        import torch
        return torch.stack(self.loss_k, dim=1)

    def bytes_per_step(self) -> int:
        b = self.fp.bytes_per_step()
        feat = sum(2 * s.numel() * 4 + s.numel() * 4 for (_c, s, _t, _d) in self.feat)
        return b["fwd"] + b["bwd"] + feat
