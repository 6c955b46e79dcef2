"""Host logic of the periodic-rescheduling experiment (tools/adapt.py, SURVEY
§8(f) F1): the two-wave rate profile (a second, higher wave) and
the thinned Poisson arrivals it drives."""
import numpy as np

from tools import adapt


def test_two_waves_second_higher():
    T = 6.0
    ts = np.linspace(0, T, 601)
    w = np.array([adapt.wave(t, T, 0.0) for t in ts])
    assert w.min() >= 0.25 - 1e-9 and w.max() <= 1.0 + 1e-9
    first = w[(ts > 0.05 * T) & (ts < 0.5 * T)].max()
    second = w[ts >= 0.5 * T].max()
    assert second > first > 0.6                          # two waves, the second higher
    # a trough between them
    assert w[(ts > 0.4 * T) & (ts < 0.55 * T)].min() < 0.35


def test_thinned_poisson_counts():
    T, peak = 4.0, [20000, 0, 3000, 0, 0, 0]
    t, m = adapt.trace(peak, T, 7)
    assert np.all(np.diff(t) >= 0) and t.min() >= 0 and t.max() < T * 1e6
    for mi, r in enumerate(peak):
        n = int((m == mi).sum())
        want = r * np.mean([adapt.wave(x, T, 0.03 * mi) for x in np.linspace(0, T, 4001)]) * T
        if r == 0:
            assert n == 0
        else:
            assert abs(n - want) < 5 * np.sqrt(want) + 0.02 * want   # mean of the thinned process
    t2, m2 = adapt.trace(peak, T, 7)
    assert np.array_equal(t, t2) and np.array_equal(m, m2)      # seeded
