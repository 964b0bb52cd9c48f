"""Pins for the oracle's counter-based generator (contract R1-R8) and digest (D1).

Every expected value here comes from something other than the oracle:
published known-answer vectors, cuRAND's own Philox routine compiled for the
host, Python big-integer / exact rational arithmetic.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import ROOT, mulhi64_bigint

GOLDEN = os.path.join(ROOT, "tests", "golden")


def _rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def test_philox_known_answer_vectors(orc):
    # R1 pinned by Random123's published KAT (tests/golden/philox4x32_10_kat.txt)
    for row in _rows("philox4x32_10_kat.txt"):
        v = [int(x, 16) for x in row if x != "->"]
        out = orc.philox4x32_10(v[0:4], v[4:6])
        assert [int(x) for x in out] == v[6:10]


def test_philox_equals_curand_routine(orc, curand_host):
    # R1 pinned by cuRAND's curand_Philox4x32_10 (library routine, host build)
    rng = np.random.default_rng(1234)
    ctr = rng.integers(0, 2**32, size=(2000, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(2000, 2), dtype=np.uint64).astype(np.uint32)
    ref = curand_host.blocks(ctr, key)
    for i in range(0, 2000, 7):
        assert list(orc.philox4x32_10(ctr[i], key[i])) == list(ref[i])


@pytest.mark.parametrize("seed,tag,t", [(42, 0x01, 0), (11, 0x01, 999), (2**40 + 3, 0x12, 0),
                                        (7, 0x11, 17)])
def test_lane_layout_against_curand(orc, curand_host, seed, tag, t):
    # R2-R4: key/counter composition and lane -> word mapping
    us = np.array([0, 1, 2, 3, 4, 5, 6, 7, 1000, 1001, 2**33 + 5, 99_999_999], dtype=np.uint64)
    ref64 = curand_host.lane64(seed, tag, us, t)
    ref32 = curand_host.lane32(seed, tag, us, t)
    for k, u in enumerate(us):
        assert orc.lane64(seed, tag, int(u), t) == int(ref64[k])
        assert orc.lane32(seed, tag, int(u), t) == int(ref32[k])


def test_mulhi64_bigint(orc):
    # R6 pinned by Python big-integer arithmetic
    rng = np.random.default_rng(5)
    xs = [0, 1, 2**64 - 1, 2**63] + [int(x) for x in rng.integers(0, 2**63, 200, dtype=np.int64)]
    for n in (1, 2, 3, 1000, 100_000_000, 2**32 + 7, 2**63):
        for x in xs:
            assert orc.mulhi64(x, n) == (x * n) >> 64
            assert 0 <= orc.mulhi64(x, n) < n


def test_bernoulli_threshold_exact(orc):
    # R7: T(p) = ceil(p * 2^32) exactly (Fraction of the double p)
    for p in (0.0, 1e-9, 0.01, 0.05, 0.1, 0.2, 1 / 3, 0.5, 0.999999, 1.0):
        exact = math.ceil(Fraction(p) * 2**32)
        assert orc.bernoulli_threshold(p) == exact
    # the values quoted in SURVEY.md 8(c) R7
    assert orc.bernoulli_threshold(0.05) == 214_748_365
    assert orc.bernoulli_threshold(0.1) == 429_496_730
    assert orc.bernoulli_threshold(0.01) == 42_949_673
    assert orc.bernoulli_threshold(0.2) == 858_993_460
    # p = 1 is always true for any 32-bit draw; p = 0 never
    assert orc.bernoulli_threshold(1.0) == 2**32 and orc.bernoulli_threshold(0.0) == 0


def test_u01_exact(orc):
    # R8: (x >> 8) * 2^-24, exact in float32, in [0, 1)
    for x in (0, 1, 255, 256, 2**31, 2**32 - 1, 0xDEADBEEF):
        assert Fraction(orc.u01(x)) == Fraction(x >> 8, 2**24)
        assert 0.0 <= orc.u01(x) < 1.0


def test_splitmix_finaliser_reference_outputs(orc):
    # D1's mix64 pinned by the splitmix64 reference outputs for seed 0
    want = [int(r[0], 16) for r in _rows("splitmix64_seed0.txt")]
    g = 0x9E3779B97F4A7C15
    got = [orc.mix64((k * g) % 2**64) for k in (1, 2, 3)]
    assert got == want


def test_digest_shard_additive_and_sensitive(orc):
    # D1 invariants: sum over shards == whole; any single change is detected
    rng = np.random.default_rng(3)
    col = rng.integers(-5, 50, size=10_001).astype(np.int32)
    whole = orc.digest(col)
    cut = [0, 17, 5000, 9999, 10_001]
    parts = sum(orc.digest(col[a:b], id0=a) for a, b in zip(cut[:-1], cut[1:])) % 2**64
    assert parts == whole
    for pos in (0, 1234, 10_000):
        c2 = col.copy()
        c2[pos] += 1
        assert orc.digest(c2) != whole
    # empty column digests to 0 (empty sum)
    assert orc.digest(np.zeros(0, np.int32)) == 0
    # uint8 columns are zero-extended: same digest as the int32 copy
    s = rng.integers(0, 3, size=999).astype(np.uint8)
    assert orc.digest(s) == orc.digest(s.astype(np.int32))


def test_round_count(orc):
    assert orc.round_count(100_000 * 10 / 2) == 500_000
    assert orc.round_count(10_000 * 8 / 2) == 40_000
    assert orc.round_count(0.01 * 100_000) == 1000
    assert orc.round_count(0.01 * 10_000) == 100
    assert orc.round_count(2.5) == 3 and orc.round_count(2.4999) == 2
