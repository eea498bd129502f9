"""GPU: the execution plan (qf::run_quant_conv's quantization, exec.hpp:
222-405) — fused and per-operator plans bit-identical, fault-injection
fallback on the GPU per-operator path, weight cache, HalfActivations, live
counters == the modeled schedule (test_exec.cpp:96-290 analogues)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from test_gpu_fwd import bits32, host, to_dev  # noqa: E402


def toy_roster(rng):
    """A small roster of (activation [C,H,W], weight [co,ci,k,k], log_w, log_a)."""
    specs = [((3, 32, 40), (8, 3, 7, 7)), ((8, 16, 20), (8, 8, 3, 3)), ((8, 16, 20), (16, 8, 3, 3)),
             ((16, 8, 10), (16, 16, 1, 1))]
    out = []
    for a, wsh in specs:
        x = rng.normal(0, 1, a).astype(np.float32)
        w = rng.normal(0, 0.3, wsh).astype(np.float32)
        lw = np.log(np.expm1(np.abs(w).reshape(wsh[0], -1).max(axis=1) / 127.0))
        la = float(np.log(np.expm1(np.abs(x).max() / 127.0)))
        out.append((x, w, lw, la))
    return out


def run(qfb, plan, roster, cuda, dtype=None, frames=1):
    import torch
    ex = qfb.ExecutionContext(plan)
    res = []
    for _ in range(frames):
        for i, (x, w, lw, la) in enumerate(roster):
            qa, qw = ex.quant_layer(i, to_dev(x, cuda, dtype), to_dev(w, cuda), lw.tolist(), la)
            res.append((host(qa), host(qw)))
    tr = ex.trace
    ex.close()
    return res, tr


def test_fused_equals_perop_and_oracle(qfb, orc, cuda):
    rng = np.random.default_rng(1)
    roster = toy_roster(rng)
    a, ta = run(qfb, qfb.ExecutionPlan(mode=qfb.MODE_FUSED), roster, cuda)
    b, tb = run(qfb, qfb.ExecutionPlan(mode=qfb.MODE_PER_OPERATOR), roster, cuda)
    for (qa1, qw1), (qa2, qw2), (x, w, lw, la) in zip(a, b, roster):
        assert np.array_equal(bits32(qa1), bits32(qa2))
        assert np.array_equal(bits32(qw1), bits32(qw2))
        _, wa = orc.fake_quantize(x, [qfb.resolve_scale(la)], 1, 1, x.size)
        _, ww = orc.fake_quantize(w, qfb.resolve_scale(lw.tolist()), 1, w.shape[0], w[0].size)
        assert np.array_equal(bits32(qa1.ravel()), bits32(wa))
        assert np.array_equal(bits32(qw1.ravel()), bits32(ww))
    # live counters == modeled schedule; ratio of quant sweeps 9:3
    assert ta.pass_count == 3 * len(roster) and tb.pass_count == 9 * len(roster)
    for tr, mode in ((ta, qfb.MODE_FUSED), (tb, qfb.MODE_PER_OPERATOR)):
        exp = [qfb.model_layer_counts(qfb.ExecutionPlan(mode=mode), x.size, w.shape[0], w[0].size)
               for x, w, _, _ in roster]
        assert tr.bytes_read == sum(e.bytes_read for e in exp)
        assert tr.bytes_written == sum(e.bytes_written for e in exp)
    assert ta.launches == 2 * len(roster) and tb.launches == 8 * len(roster)
    assert tb.peak_scratch_bytes > 0 and ta.peak_scratch_bytes == 0   # per-op reserves more


def test_fault_injection_fallback(qfb, cuda):
    rng = np.random.default_rng(2)
    roster = toy_roster(rng)
    ref, _ = run(qfb, qfb.ExecutionPlan(mode=qfb.MODE_PER_OPERATOR), roster, cuda)
    got, tr = run(qfb, qfb.ExecutionPlan(mode=qfb.MODE_FUSED, fault_inject_layer=2), roster, cuda)
    assert tr.fell_back == 1
    for (a1, w1), (a2, w2) in zip(ref, got):
        assert np.array_equal(bits32(a1), bits32(a2)) and np.array_equal(bits32(w1), bits32(w2))
    with pytest.raises(qfb.FusedPathError):
        run(qfb, qfb.ExecutionPlan(mode=qfb.MODE_FUSED, fault_inject_layer=2, fallback_enabled=False),
            roster, cuda)


def test_weight_cache(qfb, cuda):
    rng = np.random.default_rng(3)
    roster = toy_roster(rng)
    res, tr = run(qfb, qfb.ExecutionPlan(cache_weights=True), roster, cuda, frames=2)
    n = len(roster)
    assert tr.pass_count == 3 * n + 2 * n     # second frame skips the weight sweeps
    for i in range(n):
        assert np.array_equal(bits32(res[i][1]), bits32(res[n + i][1]))
        assert np.array_equal(bits32(res[i][0]), bits32(res[n + i][0]))


@pytest.mark.parametrize("f16", [False, True])
def test_half_activations(qfb, orc, cuda, f16):
    import torch
    rng = np.random.default_rng(4)
    roster = toy_roster(rng)
    roster = [(x.astype(np.float16).astype(np.float32), w, lw, -30.0) for x, w, lw, _ in roster]
    plan = qfb.ExecutionPlan(policy=qfb.POLICY_HALF_ACTIVATIONS)
    res, _ = run(qfb, plan, roster, cuda, dtype=torch.float16 if f16 else None)
    sa = qfb.resolve_scale(-30.0, None, qfb.PREC_HALF)
    assert sa == 1e-4      # stricter half-path lower bound (exec.hpp:254)
    for (qa, _), (x, _, _, _) in zip(res, roster):
        _, want = orc.fake_quantize(x, [sa], 1, 1, x.size, half=1)
        assert np.array_equal(bits32(qa.ravel()), bits32(want))
        assert np.array_equal(qa, qa.astype(np.float16).astype(np.float32))  # on the binary16 grid
