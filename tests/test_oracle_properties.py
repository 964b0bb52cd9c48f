"""T0 property tests (hypothesis on tiny N): over random inputs the
oracle's steps equal the independent cuRAND-drawn numpy re-formulations
(wealth W1-W2, SIR S2-S3), and the binned Boids step equals the brute-force
definition; invariants (conservation, S+I+R = N, monotone S and R) hold."""
import numpy as np
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from test_oracle_sir import numpy_sir_step
from test_oracle_wealth import numpy_wealth_step

SET = settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])


@SET
@given(n=st.integers(2, 60), seed=st.integers(0, 2**64 - 1), t=st.integers(0, 2**32 - 1),
       amount=st.integers(1, 3), excl=st.integers(0, 1), data=st.data())
def test_wealth_step_property(orc, curand_host, n, seed, t, amount, excl, data):
    w = np.array(data.draw(st.lists(st.integers(0, 7), min_size=n, max_size=n)), np.int32)
    got = orc.wealth_step(w, seed, t, amount=amount, exclude_self=excl)
    want, _ = numpy_wealth_step(w, seed, t, curand_host, amount=amount, exclude_self=excl)
    assert np.array_equal(got, want)
    assert got.sum() == w.sum() and (got >= 0).all()


@SET
@given(n=st.integers(2, 40), seed=st.integers(0, 2**64 - 1), t=st.integers(0, 2**32 - 1),
       beta=st.sampled_from([0.0, 0.05, 0.3, 0.9, 1.0]), gamma=st.sampled_from([0.0, 0.1, 0.5, 1.0]),
       data=st.data())
def test_sir_step_property(orc, curand_host, n, seed, t, beta, gamma, data):
    pairs = data.draw(st.lists(st.tuples(st.integers(0, n - 1), st.integers(0, n - 1)), max_size=3 * n))
    adj = [set() for _ in range(n)]
    for a, b in pairs:
        if a != b:
            adj[a].add(b)
            adj[b].add(a)
    rp = np.zeros(n + 1, np.int32)
    rp[1:] = np.cumsum([len(s) for s in adj])
    col = np.array([j for s in adj for j in sorted(s)], np.int32)
    x = np.array(data.draw(st.lists(st.integers(0, 2), min_size=n, max_size=n)), np.uint8)
    got = orc.sir_step(rp, col, x, seed, t, beta, gamma)
    want = numpy_sir_step(rp, col, x, seed, t, beta, gamma, curand_host)
    assert np.array_equal(got, want)
    assert (got[x == 2] == 2).all() and ((got == 0) <= (x == 0)).all()  # R stays R; S never reappears


@settings(max_examples=25, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(n=st.integers(1, 120), L=st.floats(20.0, 200.0), R=st.floats(1.0, 9.0), seed=st.integers(0, 2**32))
def test_boids_binned_equals_brute_property(orc, n, L, R, seed):
    P = orc.boids_params(L=L, R=R, rs=R / 3, wc=0.2, wa=0.3, ws=0.4, vmax=1.5)
    s = orc.boids_init(n, L, seed)
    a = orc.boids_step(s, P)
    b = orc.boids_step(s, P, brute=True)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert ((a[0] >= 0) & (a[0] < np.float32(L)) & (a[1] >= 0) & (a[1] < np.float32(L))).all()
