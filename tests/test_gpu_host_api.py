"""GPU parity of the host-level (value-semantics) C-ABI entry points — the
exact calls a reference user makes with host buffers (quant.hpp:136-294)."""
import ctypes
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from test_gpu_fwd import bits32  # noqa: E402


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def test_host_fwd_codes_bwd(qfb, orc, ref, cuda):
    L = qfb.lib()
    ctx = qfb.Context(0)
    cfg = qfb.QuantConfig().to_c()
    rng = np.random.default_rng(3)
    C, H, W = 32, 60, 80
    x = rng.normal(0, 1, (C, H, W)).astype(np.float32)
    up = rng.normal(0, 1, (C, H, W)).astype(np.float32)
    s = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), C))
    y = np.empty_like(x)
    qfb.check(L.qfb_fake_quantize_host(ctx.handle, 0, _p(x), _p(y), 1, C, H * W,
                                       s.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(cfg)))
    _, want = ref.fake_quantize(x, [C, H, W], s, per_channel=True)
    assert np.array_equal(bits32(y.ravel()), bits32(want))
    codes = np.empty(x.size, dtype=np.int8)
    qfb.check(L.qfb_int8_codes_host(ctx.handle, _p(x), _p(codes), 1, C, H * W,
                                    s.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(cfg)))
    _, cw = ref.int8_codes(x, [C, H, W], s, per_channel=True)
    assert np.array_equal(codes, cw)
    ls = np.log(np.expm1(s))
    dx = np.empty_like(x)
    dls = np.zeros(C)
    qfb.check(L.qfb_fake_quantize_backward_host(
        ctx.handle, 0, _p(x), _p(up), _p(dx), 1, C, H * W,
        ls.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(cfg),
        dls.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 0))
    _, wdx, wdls = ref.fq_backward(x, up, [C, H, W], ls, per_channel=True)
    assert np.array_equal(bits32(dx.ravel()), bits32(wdx))
    assert dls.tobytes() == wdls.tobytes()     # bit-identical to the reference itself
    # half path: NaN -> NonFiniteError like demote_half
    xh = x.astype(np.float16).astype(np.float32)
    xh[0, 0, 0] = np.nan
    st = L.qfb_fake_quantize_host(ctx.handle, 1, _p(xh), _p(y), 1, C, H * W,
                                  s.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(cfg))
    assert st == 4
    # bad scale -> ValueError before any compute
    s_bad = s.copy()
    s_bad[1] = 0.0
    st = L.qfb_fake_quantize_host(ctx.handle, 0, _p(x), _p(y), 1, C, H * W,
                                  s_bad.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(cfg))
    assert st == 2
    ctx.close()


@pytest.mark.parametrize("half", [0, 1])
def test_quant_pass_host_matches_reference(qfb, orc, ref, cuda, half):
    """Frame-level pipelined host pass == per-point reference calls, bitwise
    (forward outputs, d_input and scale gradients); half=1 is the
    reference's EmulatedHalf activations (inputs on the binary16 grid,
    outputs re-rounded, the half-mode scale floor in the backward)."""
    import torch
    rng = np.random.default_rng(11 + half)

    def grid(a):
        return a.astype(np.float16).astype(np.float32) if half else a
    shapes = [(3, 48, 64, 2), (32, 24, 32, 1), (32, 24, 32, 2), (64, 12, 16, 1), (7, 5, 9, 1)]
    keep, pts, checks = [], [], []
    D = ctypes.POINTER(ctypes.c_double)
    for C, H, W, n_out in shapes:
        x = torch.from_numpy(grid(rng.normal(0, 1, C * H * W).astype(np.float32))).pin_memory()
        p = qfb.CHostPoint()
        p.x = x.data_ptr()
        p.outer, p.channels, p.inner, p.n_out = 1, C, H * W, n_out
        keep.append(x)
        for k in range(n_out):
            s = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), C))
            ls = np.log(np.expm1(s))
            up = torch.from_numpy(grid(rng.normal(0, 1, C * H * W).astype(np.float32))).pin_memory()
            y = torch.empty(C * H * W).pin_memory()
            dx = torch.empty(C * H * W).pin_memory()
            dls = np.zeros(C)
            keep += [s, ls, up, y, dx, dls]
            p.s[k] = s.ctypes.data
            p.y[k] = y.data_ptr()
            p.log_s[k] = ls.ctypes.data
            p.up[k] = up.data_ptr()
            p.dx[k] = dx.data_ptr()
            p.d_log_s[k] = dls.ctypes.data
            checks.append((x.numpy(), s, ls, up.numpy(), y, dx, dls, C, H * W))
        pts.append(p)
    ctx = qfb.Context(0)
    cfg = qfb.QuantConfig().to_c()
    table = (qfb.CHostPoint * len(pts))(*pts)
    for _ in range(2):
        qfb.check(qfb.lib().qfb_quant_pass_host(ctx.handle, half, table, len(pts), ctypes.byref(cfg)))
        for x, s, ls, up, y, dx, dls, C, HW in checks:
            _, wy = ref.fake_quantize(x, [C, HW], s, half=half, per_channel=True)
            assert np.array_equal(bits32(y.numpy()), bits32(wy))
            _, wdx, wdls = ref.fq_backward(x, up, [C, HW], ls, per_channel=True, half=half)
            assert np.array_equal(bits32(dx.numpy()), bits32(wdx))
            assert dls.tobytes() == wdls.tobytes()
    ctx.close()


def _pass_table(qfb, rng, shapes):
    import torch
    keep, pts, checks = [], [], []
    for C, H, W, n_out in shapes:
        x = torch.from_numpy(rng.normal(0, 1, C * H * W).astype(np.float32)).pin_memory()
        p = qfb.CHostPoint()
        p.x = x.data_ptr()
        p.outer, p.channels, p.inner, p.n_out = 1, C, H * W, n_out
        keep.append(x)
        for k in range(n_out):
            s = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), C))
            ls = np.log(np.expm1(s))
            up = torch.from_numpy(rng.normal(0, 1, C * H * W).astype(np.float32)).pin_memory()
            y = torch.empty(C * H * W).pin_memory()
            dx = torch.empty(C * H * W).pin_memory()
            dls = np.zeros(C)
            keep += [s, ls, up, y, dx, dls]
            p.s[k], p.y[k], p.log_s[k] = s.ctypes.data, y.data_ptr(), ls.ctypes.data
            p.up[k], p.dx[k], p.d_log_s[k] = up.data_ptr(), dx.data_ptr(), dls.ctypes.data
            checks.append((x.numpy(), s, ls, up.numpy(), y, dx, dls, C, H * W))
        pts.append(p)
    return (qfb.CHostPoint * len(pts))(*pts), len(pts), checks, keep


def test_quant_pass_two_slots_in_flight(qfb, ref, cuda):
    """submit(slot 0), submit(slot 1), wait both: each slot's outputs equal
    the reference's per-point calls; a busy slot refuses a second submit."""
    rng = np.random.default_rng(21)
    shapes = [(3, 48, 64, 2), (32, 24, 32, 1), (64, 12, 16, 2)]
    t0 = _pass_table(qfb, rng, shapes)
    t1 = _pass_table(qfb, rng, shapes)
    ctx = qfb.Context(0)
    cfg = qfb.QuantConfig().to_c()
    L = qfb.lib()
    for _ in range(2):
        qfb.check(L.qfb_quant_pass_host_submit(ctx.handle, 0, t0[0], t0[1], ctypes.byref(cfg), 0))
        qfb.check(L.qfb_quant_pass_host_submit(ctx.handle, 0, t1[0], t1[1], ctypes.byref(cfg), 1))
        assert L.qfb_quant_pass_host_submit(ctx.handle, 0, t0[0], t0[1], ctypes.byref(cfg), 0) == 2
        qfb.check(L.qfb_quant_pass_host_wait(ctx.handle, 0))
        qfb.check(L.qfb_quant_pass_host_wait(ctx.handle, 1))
        for checks in (t0[2], t1[2]):
            for x, s, ls, up, y, dx, dls, C, HW in checks:
                _, wy = ref.fake_quantize(x, [C, HW], s, per_channel=True)
                assert np.array_equal(bits32(y.numpy()), bits32(wy))
                _, wdx, wdls = ref.fq_backward(x, up, [C, HW], ls, per_channel=True)
                assert np.array_equal(bits32(dx.numpy()), bits32(wdx))
                assert dls.tobytes() == wdls.tobytes()
    ctx.close()


def _pass_table_arena(qfb, rng, shapes):
    """The same table with every host buffer carved out of two pinned arenas
    in the library's copy order (inputs: x, then the upstreams; outputs: y,
    then d_input, per consumer): the pass merges contiguous copies."""
    import torch
    r16 = lambda n: (n + 3) & ~3  # noqa: E731
    n_in = sum(r16(C * H * W) * (1 + n_out) for C, H, W, n_out in shapes)
    n_out_t = sum(2 * r16(C * H * W) * n_out for C, H, W, n_out in shapes)
    a_in = torch.empty(n_in, dtype=torch.float32).pin_memory()
    a_out = torch.empty(n_out_t, dtype=torch.float32).pin_memory()
    o_in, o_out = [0], [0]

    def take(a, o, n):
        t = a[o[0]:o[0] + n]
        o[0] += r16(n)
        return t

    keep, pts, checks = [a_in, a_out], [], []
    for C, H, W, n_out in shapes:
        x = take(a_in, o_in, C * H * W)
        x.copy_(torch.from_numpy(rng.normal(0, 1, C * H * W).astype(np.float32)))
        p = qfb.CHostPoint()
        p.x = x.data_ptr()
        p.outer, p.channels, p.inner, p.n_out = 1, C, H * W, n_out
        for k in range(n_out):
            s = np.exp(rng.uniform(np.log(1e-3), np.log(0.1), C))
            ls = np.log(np.expm1(s))
            up = take(a_in, o_in, C * H * W)
            up.copy_(torch.from_numpy(rng.normal(0, 1, C * H * W).astype(np.float32)))
            y = take(a_out, o_out, C * H * W)
            dx = take(a_out, o_out, C * H * W)
            dls = np.zeros(C)
            keep += [s, ls, dls]
            p.s[k], p.y[k], p.log_s[k] = s.ctypes.data, y.data_ptr(), ls.ctypes.data
            p.up[k], p.dx[k], p.d_log_s[k] = up.data_ptr(), dx.data_ptr(), dls.ctypes.data
            checks.append((x.numpy(), s, ls, up.numpy(), y, dx, dls, C, H * W))
        pts.append(p)
    return (qfb.CHostPoint * len(pts))(*pts), len(pts), checks, keep


def test_quant_pass_merged_copies(qfb, ref, cuda):
    """Host buffers laid out contiguously in copy order (merged DMA copies,
    both slots in flight): the same bits as the reference's per-point calls."""
    rng = np.random.default_rng(23)
    shapes = [(3, 48, 64, 2), (32, 24, 32, 1), (64, 12, 16, 2), (8, 40, 40, 1)]
    t0 = _pass_table_arena(qfb, rng, shapes)
    t1 = _pass_table_arena(qfb, rng, shapes)
    ctx = qfb.Context(0)
    cfg = qfb.QuantConfig().to_c()
    L = qfb.lib()
    for _ in range(2):
        qfb.check(L.qfb_quant_pass_host_submit(ctx.handle, 0, t0[0], t0[1], ctypes.byref(cfg), 0))
        qfb.check(L.qfb_quant_pass_host_submit(ctx.handle, 0, t1[0], t1[1], ctypes.byref(cfg), 1))
        qfb.check(L.qfb_quant_pass_host_wait(ctx.handle, 0))
        qfb.check(L.qfb_quant_pass_host_wait(ctx.handle, 1))
        for checks in (t0[2], t1[2]):
            for x, s, ls, up, y, dx, dls, C, HW in checks:
                _, wy = ref.fake_quantize(x, [C, HW], s, per_channel=True)
                assert np.array_equal(bits32(y.numpy()), bits32(wy))
                _, wdx, wdls = ref.fq_backward(x, up, [C, HW], ls, per_channel=True)
                assert np.array_equal(bits32(dx.numpy()), bits32(wdx))
                assert dls.tobytes() == wdls.tobytes()
    ctx.close()
