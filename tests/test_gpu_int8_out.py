"""f2: int8 code emission from the fused multi-point
forward (QFB_FLAG_INT8_OUT) — bitwise equal to int8_codes (quant.hpp:174-207)
of the CPU oracle, on the TMA, vector and scalar paths, f32 and f16, with
per-channel scales and two consumers per point."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run_multi(q, cuda, xs, scales, dtype, offset=0):
    import torch
    tdt = torch.float32 if dtype == 0 else torch.float16
    keep, descs, outs = [], [], []
    for x, ss in zip(xs, scales):
        C = x.shape[0]
        base = torch.empty(x.size + 8, dtype=tdt, device=cuda)
        xd = base[offset:offset + x.size]
        xd.copy_(torch.from_numpy(x.ravel()).to(tdt))
        d = q.CFqDesc()
        d.x = xd.data_ptr()
        d.outer, d.channels, d.inner = 1, C, x.size // C
        d.n_out, d.q_max, d.flags = len(ss), 127, 0x4
        ys = []
        for k, s in enumerate(ss):
            st = torch.from_numpy(np.asarray(s, dtype=np.float32)).to(cuda)
            y = torch.empty(x.size + 16, dtype=torch.int8, device=cuda)[offset:offset + x.size]
            d.y[k], d.scale[k] = y.data_ptr(), st.data_ptr()
            ys.append(y)
            keep.append(st)
        keep += [base, xd]
        outs.append(ys)
        descs.append(d)
    table = (q.CFqDesc * len(descs))(*descs)
    q.check(q.lib().qfb_fq_fwd_multi(q.default_context(0).handle, dtype, table, len(descs)))
    torch.cuda.synchronize()
    return [[y.cpu().numpy() for y in ys] for ys in outs]


@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("offset", [0, 1])   # 1 element: unaligned -> scalar path
def test_int8_emission_matches_oracle(qfb, orc, cuda, dtype, offset):
    rng = np.random.default_rng(7 + dtype + 10 * offset)
    shapes = [(3, 48, 64), (32, 24, 32), (64, 12, 16), (5, 7, 3)]
    xs, scales = [], []
    for i, sh in enumerate(shapes):
        x = rng.normal(0, 2, sh).astype(np.float32)
        x.ravel()[:6] = [0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45]
        if dtype == 1:
            x = x.astype(np.float16).astype(np.float32)
        xs.append(x)
        k = 2 if i % 2 == 0 else 1
        scales.append([np.exp(rng.uniform(np.log(1e-3), np.log(0.1), sh[0])).astype(np.float32)
                       for _ in range(k)])
    got = run_multi(qfb, cuda, xs, scales, dtype, offset)
    for x, ss, ys in zip(xs, scales, got):
        C = x.shape[0]
        for s, y in zip(ss, ys):
            st, want = orc.int8_codes(x, s.astype(np.float64), 1, C, x.size // C)
            assert st == 0
            assert np.array_equal(y, want)
