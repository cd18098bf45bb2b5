"""Online rolling-window driver (BASELINE configs[4])."""
import numpy as np
import pytest

import paper_2504_14966_b200 as S
from paper_2504_14966_b200 import online as O


def test_stream_is_deterministic_and_poisson():
    a = O.make_stream(4000, rate_per_s=2.0, seed=3)
    b = O.make_stream(4000, rate_per_s=2.0, seed=3)
    assert np.array_equal(a.arrival_ms, b.arrival_ms) and np.array_equal(a.pred_out, b.pred_out)
    gaps = np.diff(a.arrival_ms)
    assert abs(gaps.mean() - 500.0) < 25.0  # mean inter-arrival 1 / rate
    w = S.generate_mixed(4000, 3)  # lengths are the reference generator's
    assert np.array_equal(a.input_len, w.arrays["in_len"])


def test_fcfs_completes_every_request_and_matches_a_direct_simulation():
    s = O.make_stream(300, rate_per_s=0.5, seed=1)
    r = O.run_online(s, "fcfs", n_instances=2, window_ms=5000.0)
    assert r.n == 300 and 0 < r.n_met <= 300 and r.total_latency_ms > 0
    # single instance, one huge window: FCFS = arrival-order greedy batches back to back
    s1 = O.make_stream(40, rate_per_s=1000.0, seed=2)
    r1 = O.run_online(s1, "fcfs", n_instances=1, window_ms=1e12, max_batch=4)
    c = S.table_coefficients()
    t = max(0.0, np.ceil(s1.arrival_ms[-1] / 1e12) * 1e12)  # window that holds every arrival
    n_met = 0
    order = list(range(40))
    for k in range(0, 40, 4):
        b = order[k:k + 4]
        start = t + 0.1
        li, lo = s1.input_len[b].astype(float), s1.true_out[b].astype(float)
        pf, dec = O.prefill_ms(c, len(b), li), O.decode_total_ms(c, len(b), li, lo)
        for j, i in enumerate(b):
            if s1.cls[i] == 0:
                n_met += start + pf[j] + dec[j] - s1.arrival_ms[i] <= 30000.0
            else:
                n_met += (start + pf[j] - s1.arrival_ms[i] <= 10000.0) and dec[j] / lo[j] <= 50.0
        t = start + (pf + dec).max()
    assert r1.n_met == n_met


def test_custom_planner_and_devices():
    """A caller's planner plugs in per window (here the FCFS rule itself: identical result)."""
    s = O.make_stream(400, rate_per_s=0.6, seed=5)
    ref = O.run_online(s, "fcfs", n_instances=3, window_ms=4000.0)
    fcfs_rule = lambda st, ids, start: O._plan_fcfs(st, ids, 4)[0]  # noqa: E731
    got = O.run_online(s, "custom", n_instances=3, window_ms=4000.0, planner=fcfs_rule, devices=(0, 1))
    assert (got.n, got.n_met, got.total_latency_ms, got.windows) == (ref.n, ref.n_met, ref.total_latency_ms,
                                                                      ref.windows)
    with pytest.raises(ValueError):
        O.run_online(s, "custom", n_instances=2)


@pytest.mark.parametrize("n_inst,window,mb,gap,maxw", [(3, 4000.0, 4, 0.1, None), (2, 1500.0, 8, 0.0, None),
                                                       (5, 7000.0, 2, 0.5, 6)])
def test_native_driver_matches_the_python_loop(n_inst, window, mb, gap, maxw):
    """slosched_run_online (csrc/online.cpp) and the Python loop agree on FCFS, request for request."""
    s = O.make_stream(600, rate_per_s=0.8 * n_inst * O.service_rate_per_s(), seed=11)
    kw = dict(n_instances=n_inst, window_ms=window, max_batch=mb, dispatch_gap_ms=gap, max_windows=maxw)
    nat = O.run_online(s, "fcfs", **kw)
    py = O._run_online_py(s, "fcfs", **kw)
    assert (nat.n, nat.n_met, nat.windows, nat.decisions) == (py.n, py.n_met, py.windows, py.decisions)
    assert nat.total_latency_ms == pytest.approx(py.total_latency_ms, rel=1e-12)
    assert len(nat.overhead_ms) == nat.windows


@pytest.mark.gpu
def test_online_sa_beats_fcfs():
    mu = O.service_rate_per_s()
    s = O.make_stream(1500, rate_per_s=0.9 * 2 * mu, seed=4)
    sa = O.run_online(s, "sa", n_instances=2, window_ms=5000.0, budget_ms=3.0, chains=1024)
    fc = O.run_online(s, "fcfs", n_instances=2, window_ms=5000.0)
    assert sa.n == fc.n == 1500
    assert sa.n_met >= fc.n_met
    assert max(sa.overhead_ms) < 1000.0
    py = O._run_online_py(s, "sa", n_instances=2, window_ms=5000.0, budget_ms=3.0, chains=1024)
    assert py.n == 1500 and py.n_met >= fc.n_met


def test_native_driver_rejects_bad_input():
    import numpy as np

    from paper_2504_14966_b200.slosched import DataError
    s = O.make_stream(50, rate_per_s=0.5, seed=2)
    with pytest.raises(DataError):
        O.run_online(s, "fcfs", n_instances=2, max_batch=0)
    with pytest.raises(DataError):
        O.run_online(s, "fcfs", n_instances=0)
    bad = O.Stream(**{**s.__dict__, "arrival_ms": np.asarray(s.arrival_ms)[::-1].copy()})
    with pytest.raises(DataError):
        O.run_online(bad, "fcfs", n_instances=2)


@pytest.mark.gpu
def test_cpp_online_example():
    """examples/online_example.cpp: the online driver through the C++ API (GPU chains vs FCFS)."""
    import os
    import subprocess

    from conftest import ROOT
    exe = os.path.join(ROOT, "examples", "_build", "online_example")
    assert os.path.exists(exe), "examples are built by python -m paper_2504_14966_b200.build"
    out = subprocess.run([exe, "1200", "2"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 3 and "FAIL" not in out.stdout
