"""DPVO front-end quant pass: every activation quant point of the two
BasicEncoder4 encoders (fnet, inet) for a batch of 480x640 frames, run as ONE
fused forward launch and ONE backward launch through the C-ABI tables.

This is the B200 counterpart of the quant portion of the reference's
front-end walk (exec.hpp:416-460 run_frontend / frontend.hpp:170-258
forward_train + backward_train): per quant point the activation fake-quant
forward (exec.hpp:353-361) and the scale-only backward
(frontend.hpp:226-229 -> quant.hpp:261-294). The convolutions themselves are
out of scope (cuDNN territory).

The quant-point catalogue and byte model live in ``shapes`` (pure Python,
re-exported here).
"""
from __future__ import annotations

import ctypes

import os

import numpy as np

from . import BWD_ROWS, CBwdDesc, CChainDesc, CFqDesc, F16, F32, Context, check, lib, scale_grad_factors
from .shapes import (ACT_GELU, ACT_NONE, ACT_RELU, H, W, ChainPoint, QuantPoint,  # noqa: F401
                     dpvo_quant_points, frame_bytes, window_chain_points)



# diagnostic A/B knob: extra QFB_FLAG_* bits on the forward descriptors
# (e.g. QFB_FWD_EXTRA_FLAGS=2: evict-first loads/stores); results unchanged
_FWD_EXTRA_FLAGS = int(os.environ.get("QFB_FWD_EXTRA_FLAGS", "0"))

class FrontendQuantPass:
    """Device buffers + C-ABI descriptor tables for `frames` frames of the
    DPVO activation set, per-channel scales (log-uniform [1e-3, 0.1],
    SURVEY §8d C2). `sets` independent input sets rotate so consecutive
    steps never hit L2-resident inputs."""

    def __init__(self, ctx: Context, frames: int = 1, dtype: str = "f32", sets: int = 1,
                 seed: int = 1, device=None, h: int = H, w: int = W, int8_out: bool = False,
                 grads_out=None, rows_out=None, frame_offset: int = 0):
        """int8_out: the forward emits the int8 codes of every quant point
        (QFB_FLAG_INT8_OUT, 1 byte per element) instead of the
        fake-quant values; the backward is unchanged.
        grads_out: float64 [n_grad] receiving the frame-order fold of the
        scale gradients (the finisher folds the frames, frontend.hpp:222-228).
        rows_out: float64 [frames, n_grad] receiving one gradient row per
        frame instead (QFB_BWD_ROWS), for the multi-GPU exchange, which
        gathers the rows of every rank and folds them in global frame order.
        frame_offset: global index of this pass's first frame: every frame's
        data depends only on its global index (rng.hpp counter offsets), so
        a frame shard on rank r holds exactly the frames a single GPU would."""
        import torch
        self.ctx = ctx
        self.frames = frames
        self.frame_offset = frame_offset
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
        self.n_grad = n_grad
        self.dls_flat = (grads_out if grads_out is not None
                         else torch.zeros(n_grad, dtype=torch.float64, device=dev))
        assert self.dls_flat.numel() == n_grad and self.dls_flat.dtype == torch.float64
        self.rows = rows_out
        if rows_out is not None:
            assert tuple(rows_out.shape) == (frames, n_grad) and rows_out.dtype == torch.float64
            assert rows_out.is_contiguous()
        self.goff = []
        goff = 0
        s64_all, chain_all = [], []
        for p, _ in self.consumers:
            s = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), p.channels))
            ls = np.log(np.expm1(s))
            s64, chain = scale_grad_factors(ls.tolist())
            self.log_s.append(ls)
            s64_all += s64
            chain_all += chain
            self.dls.append(self.dls_flat[goff:goff + p.channels])
            self.goff.append(goff)
            goff += p.channels
        # resolved scales of every consumer, flat (one device resolve or one
        # upload refreshes them all): float32 for the forward, double s and
        # chain factor for the backward (quant.hpp:138,162 / 241-244)
        self.s64_flat = torch.tensor(s64_all, dtype=torch.float64, device=dev)
        self.chain_flat = torch.tensor(chain_all, dtype=torch.float64, device=dev)
        self.s32_flat = torch.tensor(np.array(s64_all, dtype=np.float64).astype(np.float32), device=dev)
        for ci, (p, _) in enumerate(self.consumers):
            g0 = self.goff[ci]
            self.s32.append(self.s32_flat[g0:g0 + p.channels])
            self.fac.append((self.s64_flat[g0:g0 + p.channels], self.chain_flat[g0:g0 + p.channels]))
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
                                     seed + 1000 * si, pi, frame_offset * p.numel, 1, 1.0, 0.0))
                xs.append(t)
            ups = []
            for ci, (p, _) in enumerate(self.consumers):
                t = torch.empty((frames, p.channels, p.height, p.width), dtype=tdt, device=dev)
                check(L.qfb_fill_rng(ctx.handle, self.dtype_code, t.data_ptr(), t.numel(),
                                     seed + 1000 * si + 500, ci, frame_offset * p.numel, 1, 1.0, 0.0))
                ups.append(t)
            self.sets.append(self._tables(xs, ups))
        # size the backward workspace now, so the first call may be captured
        for st in self.sets:
            check(L.qfb_fq_bwd_reserve(ctx.handle, self.dtype_code, st["bwd"], st["nb"]))
        ctx.sync()

    def _tables(self, xs, ups):
        fwd, bwd = [], []
        ci = 0
        for pi, p in enumerate(self.points):
            d = CFqDesc()
            d.x = xs[pi].data_ptr()
            d.outer, d.channels, d.inner = self.frames, p.channels, p.inner
            d.n_out, d.q_max, d.flags = len(p.consumers), 127, (0x4 if self.int8_out else 0) | _FWD_EXTRA_FLAGS
            for k in range(len(p.consumers)):
                d.y[k] = self.y[ci + k].data_ptr()
                d.scale[k] = self.s32[ci + k].data_ptr()
            fwd.append(d)
            for k in range(len(p.consumers)):
                b = CBwdDesc()
                b.x, b.up, b.dx = xs[pi].data_ptr(), ups[ci + k].data_ptr(), self.dx[ci + k].data_ptr()
                b.scale64 = self.fac[ci + k][0].data_ptr()
                b.chain = self.fac[ci + k][1].data_ptr()
                b.outer, b.channels, b.inner = self.frames, p.channels, p.inner
                if self.rows is None:
                    b.d_log_s = self.dls[ci + k].data_ptr()
                    b.q_max, b.accumulate = 127, 0
                else:
                    b.d_log_s = self.rows.data_ptr() + 8 * self.goff[ci + k]
                    b.q_max, b.accumulate, b.row_stride = 127, BWD_ROWS, self.n_grad
                bwd.append(b)
            ci += len(p.consumers)
        ft = (CFqDesc * len(fwd))(*fwd)
        bt = (CBwdDesc * len(bwd))(*bwd)
        return {"x": xs, "up": ups, "fwd": ft, "nf": len(fwd), "bwd": bt, "nb": len(bwd)}

    def set_log_scales(self, log_s_flat) -> None:
        """Resolve every consumer's scales from a flat float64 vector of log
        scales on the HOST (glibc, bitwise the reference's resolve_scale /
        chain factors, quant.hpp:95-109, 241-244) and upload them."""
        import torch
        ls = np.ascontiguousarray(log_s_flat, dtype=np.float64)
        s64, chain = scale_grad_factors(ls.tolist())
        self.s64_flat.copy_(torch.tensor(s64, dtype=torch.float64))
        self.chain_flat.copy_(torch.tensor(chain, dtype=torch.float64))
        self.s32_flat.copy_(torch.tensor(np.array(s64, dtype=np.float64).astype(np.float32)))

    def resolve_on_device(self, log_s_dev, ctx: Context = None) -> None:
        """The same on the device (qfb_resolve_scales_dev, one launch,
        capturable): CUDA's double log1p/exp may differ from glibc by an
        ulp, so scales resolved this way are within 2 ulp of the host's
        (DESIGN.md §2), not bitwise."""
        from . import QuantConfig
        cfg = QuantConfig().to_c()
        check(lib().qfb_resolve_scales_dev((ctx or self.ctx).handle, log_s_dev.data_ptr(), self.n_grad,
                                           ctypes.byref(cfg), 0, self.s32_flat.data_ptr(),
                                           self.s64_flat.data_ptr(), self.chain_flat.data_ptr()))

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

class LocalFold:
    """Exchange of a single-GPU step: the per-frame gradient rows folded in
    frame order (qfb_fold_rows, one launch, capturable)."""

    def __init__(self, ctx: Context):
        self.ctx = ctx

    def __call__(self, rows, out) -> None:
        check(lib().qfb_fold_rows(self.ctx.handle, rows.data_ptr(), rows.shape[0], rows.shape[1], None,
                                  out.data_ptr()))


class NcclGatherFold:
    """The multi-GPU exchange on the product path: this rank's per-frame
    gradient rows [F, n] all-gathered over NCCL and folded in global frame
    order, in one C-ABI call (qfb_gather_fold_scale_grads = ncclAllGather +
    qfb_fold_rows on the context stream, capturable into the step's CUDA
    graph). Bit-identical to the single-GPU frame-order accumulation
    (distill.hpp:249-250, frontend.hpp:222-228) at every GPU count."""

    def __init__(self, ctx: Context, comm, rows_per_rank: int, n: int, device=None):
        import torch
        self.ctx, self.comm, self.F, self.n = ctx, comm, rows_per_rank, n
        dev = device if device is not None else torch.device("cuda", ctx.device)
        self.gathered = torch.empty((comm.nranks * rows_per_rank, n), dtype=torch.float64, device=dev)

    def __call__(self, rows, out) -> None:
        assert tuple(rows.shape) == (self.F, self.n)
        check(lib().qfb_gather_fold_scale_grads(self.ctx.handle, self.comm.handle, rows.data_ptr(), self.F,
                                                self.n, self.gathered.data_ptr(), None, out.data_ptr()))


class GlooGatherFold:
    """Test-only exchange for ranks sharing one GPU (NCCL refuses two ranks
    on one device): the rows go through torch.distributed gloo on the host,
    then the same device fold. Not capturable."""

    def __init__(self, ctx: Context):
        self.ctx = ctx

    def __call__(self, rows, out) -> None:
        import torch
        import torch.distributed as dist
        ws = dist.get_world_size()
        host = rows.cpu()
        parts = [torch.empty_like(host) for _ in range(ws)]
        dist.all_gather(parts, host)
        allr = torch.cat(parts).to(rows.device)
        LocalFold(self.ctx)(allr, out)


class QatStep:
    """One scale-only QAT step over a chunk of `total_frames` frames, of
    which this process holds `frames` starting at global frame
    `frame_offset` (all of them on one GPU). Every piece is a qfb launch:

      forward_backward(): fused FQ forward of every quant point (1 launch),
        the distillation loss of every frame's fnet / inet pair (upstream
        scaled by 1/chunk_len, distill.hpp:241-248), the scale-only backward
        (1 launch + finisher) leaving ONE gradient row per frame;
      exchange():  the rows folded in global frame order (LocalFold on one
        GPU; NcclGatherFold across GPUs) into the gradient vector;
      optimizer(): Adam with the step counter on the device (DeviceAdam),
        skipped on non-finite gradients or losses (distill.hpp:254-279).

    Adam runs only after the exchange, so every rank applies the same
    update to the same replicated scales (bitwise equal replicas, equal to
    the single-GPU step). With resolve="device" and a capturable exchange
    the whole step replays as one CUDA graph and successive replays are
    successive steps; resolve="host" (default) resolves the scales with the
    host libm between steps, bit-identical to the reference."""

    def __init__(self, ctx: Context, frames: int = 64, dtype: str = "f32", seed: int = 21, device=None,
                 h: int = H, w: int = W, lambda_cos: float = 1.0, lr: float = 5e-3,
                 n_weight_scales: int = 592, frame_offset: int = 0, total_frames: int = None,
                 exchange=None, resolve: str = "host"):
        import torch
        from . import DeviceAdam
        self.ctx = ctx
        self.frames = frames
        self.seed = seed
        self.frame_offset = frame_offset
        self.total_frames = total_frames or frames
        self.lam = lambda_cos
        self.lr = lr
        dev = device if device is not None else torch.device("cuda", ctx.device)
        n_act = sum(p.channels * len(p.consumers) for p in dpvo_quant_points(h, w))
        self.n_act = n_act
        self.n_params = n_act + n_weight_scales
        # the exchange writes the folded scale gradients into the optimizer's vector
        self.grads = torch.zeros(self.n_params, dtype=torch.float64, device=dev)
        self.rows = torch.zeros((frames, n_act), dtype=torch.float64, device=dev)
        self.fp = FrontendQuantPass(ctx, frames=frames, dtype=dtype, sets=1, seed=seed, device=dev, h=h, w=w,
                                    rows_out=self.rows, frame_offset=frame_offset)
        h4, w4 = h // 4, w // 4
        L = lib()
        # synthetic student / teacher encoder outputs per frame (fnet 128, inet 384 channels)
        self.feat = []
        for k, c in enumerate((128, 384)):
            t = [torch.empty((frames, c, h4, w4), dtype=torch.float32, device=dev) for _ in range(2)]
            for j, tt in enumerate(t):
                check(L.qfb_fill_rng(ctx.handle, F32, tt.data_ptr(), tt.numel(), seed + 17, 10 * k + j,
                                     frame_offset * c * h4 * w4, 1, 1.0, 0.0))
            self.feat.append((c, t[0], t[1], torch.empty_like(t[0])))
        # per pair (fnet, inet): [frames][mse, cos]
        self.loss_flat = torch.zeros((2, frames, 2), dtype=torch.float64, device=dev)
        # flattened trainable scales: the activation scales of the pass + weight scales
        self.params = torch.empty(self.n_params, dtype=torch.float64, device=dev)
        self.params[:n_act] = torch.from_numpy(np.concatenate(self.fp.log_s)).to(dev)
        self.params[n_act:] = -4.0
        self.adam = DeviceAdam(self.params, lr=lr)
        self.exchange_fn = exchange if exchange is not None else LocalFold(ctx)
        if resolve not in ("host", "device"):
            raise ValueError("resolve must be 'host' or 'device'")
        self.resolve = resolve
        ctx.sync()
        torch.cuda.synchronize(dev)

    @property
    def m(self):
        return self.adam.m

    @property
    def v(self):
        return self.adam.v

    def resolve_scales(self) -> None:
        """Scales of this step from the current log scales (forward_train
        resolves them per layer each step, frontend.hpp:103-120): on the host
        (glibc, bitwise, needs a sync: eager steps) or on the device (one
        capturable launch, within 2 ulp of glibc)."""
        if self.resolve == "device":
            self.fp.resolve_on_device(self.params[:self.n_act], ctx=self.ctx)
        else:
            self.ctx.sync()
            self.fp.set_log_scales(self.params[:self.n_act].cpu().numpy())

    def forward_backward(self) -> None:
        """fwd (1 launch) -> per-frame distill loss (2 pairs) -> bwd (1
        launch + finisher): one gradient row per frame in self.rows."""
        from . import _lib, _vp
        self.fp.forward(0)
        inv = 1.0 / self.total_frames
        for k, (c, s, t, d) in enumerate(self.feat):
            # every frame's pair_loss in one batched call (per-frame trees)
            hw = s.shape[2] * s.shape[3]
            check(_lib.qfb_distill_batch(self.ctx.handle, _vp(s.data_ptr()), _vp(t.data_ptr()), self.frames, c,
                                         hw, self.lam, inv, _vp(d.data_ptr()),
                                         _vp(self.loss_flat[k].data_ptr())))
        self.fp.backward(0)

    def exchange(self) -> None:
        """Rows of the whole chunk (all ranks) folded in frame order into
        the activation part of the gradient vector."""
        self.exchange_fn(self.rows, self.grads[:self.n_act])

    def optimizer(self) -> None:
        self.adam.step(self.grads, loss=self.loss_flat, ctx=self.ctx)

    def run(self) -> None:
        self.resolve_scales()
        self.forward_backward()
        self.exchange()
        self.optimizer()

    def losses(self):
        """[frames, 2 pairs, (mse, cos)] of the last run."""
        return self.loss_flat.permute(1, 0, 2)

    def bytes_per_step(self) -> int:
        b = self.fp.bytes_per_step()
        feat = sum(2 * s.numel() * 4 + s.numel() * 4 for (_c, s, _t, _d) in self.feat)
        return b["fwd"] + b["bwd"] + feat
