"""CPU: the execution plan's modeled counters equal an independent schedule
walker restated from the reference's test (test_exec.cpp:23-92) — without
the conv pass, which stays with the caller — and reproduce the reference's
pinned direction-of-effect properties (pass ratio, bytes >= 2x;
test_exec.cpp:96-149)."""
import pytest

import paper_2511_12653_b200 as q

# DPVO encoder roster (22 convs): (n_act, c_out, per) per quant point
H, W = 480, 640


def dpvo_roster():
    r = []
    for _enc in range(2):
        r.append((3 * H * W, 32, 3 * 7 * 7))                       # conv1
        for _ in range(4):
            r.append((32 * H // 2 * W // 2, 32, 32 * 9))           # layer1
        r.append((32 * H // 2 * W // 2, 64, 32 * 9))               # l2b1 conv1
        r.append((32 * H // 2 * W // 2, 64, 32))                   # l2b1 down
        for _ in range(3):
            r.append((64 * H // 4 * W // 4, 64, 64 * 9))           # l2b1 conv2, l2b2
        r.append((64 * H // 4 * W // 4, 128, 64))                  # conv2 (fnet 128 / inet 384)
    return r


def walker(roster, per_operator):
    """test_exec.cpp:31-92 sweep rules minus the conv sweep."""
    passes = rd = wr = 0

    def sweep(a, b):
        nonlocal passes, rd, wr
        passes += 1
        rd += a
        wr += b
    for na, co, per in roster:
        nw = co * per
        sweep(4 * (co + 1), 4 * (co + 1))
        if per_operator:
            sweep(4 * na + 4, 4 * na)
            sweep(4 * na, 4 * na)
            sweep(4 * na, 4 * na)
            sweep(4 * na + 4, 4 * na)
            sweep(4 * (nw + co), 4 * nw)
            sweep(4 * nw, 4 * nw)
            sweep(4 * nw, 4 * nw)
            sweep(4 * (nw + co), 4 * nw)
        else:
            sweep(4 * na + 4, 4 * na)
            sweep(4 * (nw + co), 4 * nw)
    return passes, rd, wr


def model(roster, plan, cached=False, fault=None):
    p = r = w = 0
    fell = 0
    for i, (na, co, per) in enumerate(roster):
        t = q.model_layer_counts(plan, na, co, per, cached, fault == i)
        p += t.pass_count
        r += t.bytes_read
        w += t.bytes_written
        fell |= t.fell_back
    return p, r, w, fell


@pytest.mark.parametrize("mode", [q.MODE_PER_OPERATOR, q.MODE_FUSED])
def test_counters_match_schedule_walker(mode):
    roster = dpvo_roster()
    p, r, w, _ = model(roster, q.ExecutionPlan(mode=mode))
    assert (p, r, w) == walker(roster, mode == q.MODE_PER_OPERATOR)


def test_pass_ratio_and_bytes():
    roster = dpvo_roster()
    a = model(roster, q.ExecutionPlan(mode=q.MODE_PER_OPERATOR))
    b = model(roster, q.ExecutionPlan(mode=q.MODE_FUSED))
    # quant sweeps per layer: 9 vs 3 (the reference's 10 vs 4 adds the conv)
    assert a[0] == 9 * len(roster) and b[0] == 3 * len(roster)
    assert (a[0] + len(roster)) * 2 == (b[0] + len(roster)) * 5   # test_exec.cpp:145: ratio 2.5 with conv
    assert a[1] + a[2] >= 2 * (b[1] + b[2])


def test_fallback_and_cache_counters():
    roster = dpvo_roster()
    plan = q.ExecutionPlan(mode=q.MODE_FUSED, fault_inject_layer=3)
    p, r, w, fell = model(roster, plan, fault=3)
    assert fell == 1
    assert p == 3 * len(roster) + 6          # layer 3 ran per-operator
    strict = q.ExecutionPlan(mode=q.MODE_FUSED, fallback_enabled=False)
    with pytest.raises(q.FusedPathError):
        q.model_layer_counts(strict, 10, 2, 3, False, True)
    # weight cache: the second frame skips every weight sweep
    full = model(roster, q.ExecutionPlan(cache_weights=True))[0]
    cached = model(roster, q.ExecutionPlan(cache_weights=True), cached=True)[0]
    assert full - cached == len(roster)
