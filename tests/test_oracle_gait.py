"""Pins for computeContactSequence (O7, reading L22).

The Q0.32 integer schedule is checked against the paper's real-valued
definition frac(phi0 + f j dt + offset_i) < D_f evaluated in exact rational
arithmetic, against T_st / T_sw, and against worked values."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2403_11383_b200.workloads import base_config

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_worked_increments(orc):
    # exact rationals: round(f * dt * 2^32) with f, dt decimal
    for f, want in [("1.3", None), ("2.0", None), ("2.4", None)]:
        exact = Fraction(f) * Fraction("0.02") * 2 ** 32
        assert orc.phase_inc(float(f), 0.02) == round(exact)
    assert orc.phase_inc(1.3, 0.02) == 111669150
    assert orc.phase_inc(2.0, 0.02) == 171798692
    assert orc.phase_inc(2.4, 0.02) == 206158430
    assert orc.stance_threshold(0.65) == 2791728742


def _cfg(duty, offsets=(0.0, 0.5, 0.5, 0.0), H=12, dt=0.02):
    # exact decimal config (no binary32 rounding) for comparison with rationals
    c = base_config(horizon=H)
    c.update(duty_factor=duty, phase_offset=list(offsets), dt=dt)
    return c


def test_worked_schedule(orc):
    c = _cfg(0.65)
    for f, fr_swing in [(1.3, range(6, 12)), (2.0, range(4, 12)), (2.4, range(4, 11))]:
        d = orc.contact_sequence(c, 0, f)
        assert d[:, 0].all() and d[:, 3].all()                 # FL, RR stance all 12 steps
        for j in range(12):
            exp = 0 if j in fr_swing else 1
            assert d[j, 1] == exp and d[j, 2] == exp, (f, j)   # FR, RL


def test_full_stance_and_trot_complementarity(orc):
    c1 = _cfg(1.0)
    for f in (1.3, 2.0, 2.4):
        for ph in (0, 12345, 0xFFFFFFFF, 0x80000000):
            assert orc.contact_sequence(c1, ph, f).all()       # D_f = 1: always stance
    c = _cfg(0.5)
    rng = np.random.default_rng(3)
    for ph in rng.integers(0, 2 ** 32, 50):
        d = orc.contact_sequence(c, int(ph), 2.0)
        assert np.all(d[:, 0] + d[:, 1] == 1) and np.all(d[:, 2] + d[:, 3] == 1)


def test_duty_factor_fraction_and_timing():
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["gait_timing"]
    f, Df = g["f_s"], g["D_f"]
    assert abs(Df / f - g["T_st"]) < 1e-15 and abs((1 - Df) / f - g["T_sw"]) < 1e-15


@pytest.mark.parametrize("f", [1.3, 2.0, 2.4])
def test_duty_fraction_over_cycle(orc, f):
    # sample one whole cycle finely: the stance fraction equals D_f within one sample
    n = 1000
    dt = 1.0 / (f * n)
    c = _cfg(0.65, H=n, dt=dt)
    d = orc.contact_sequence(c, 0, f)
    for i in range(4):
        assert abs(d[:, i].sum() - 0.65 * n) <= 1.0 + 1e-9


def test_matches_exact_rational_definition(orc):
    rng = np.random.default_rng(4)
    H = 24
    mism = 0
    for trial in range(300):
        Df = [0.5, 0.6, 0.65, 0.75][trial % 4]
        f = [1.3, 2.0, 2.4][trial % 3]
        c = _cfg(Df, H=H)
        ph = int(rng.integers(0, 2 ** 32))
        d = orc.contact_sequence(c, ph, f)
        for j in range(H):
            for i, off in enumerate(c["phase_offset"]):
                x = Fraction(ph, 2 ** 32) + Fraction(str(f)) * j * Fraction("0.02") + Fraction(str(off))
                fr = x - (x.numerator // x.denominator)
                want = 1 if fr < Fraction(str(Df)) else 0
                # Q0.32 rounding may only flip a flag within (j+1) 2^-32 of a boundary
                near = min(abs(fr - Fraction(str(Df))), fr, 1 - fr) <= Fraction(j + 2, 2 ** 32)
                if d[j, i] != want:
                    assert near
                    mism += 1
    assert mism == 0


def test_periodicity(orc):
    c = _cfg(0.65, H=12)
    # advancing the phase by exactly one cycle (2^32) is the identity
    for ph in (0, 7, 2 ** 31 + 5):
        a = orc.contact_sequence(c, ph, 2.4)
        b = orc.contact_sequence(c, (ph + 2 ** 32) & 0xFFFFFFFF, 2.4)
        assert np.array_equal(a, b)
