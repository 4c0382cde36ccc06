"""Desk-scale closed-loop trend checks.  PARITY UNPINNED: the paper's
Fig. 4 and Table I come from MuJoCo / hardware runs of a full robot; here the
plant is the SRBD of Eq. 1 and only the qualitative trends are checked
("reproduces the ordering (adaptive > fixed), not the absolute
numbers").  The loop is deterministic (counter RNG, ordered reductions), so
these runs are reproducible bit for bit on a given build.
"""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_11383_b200 import binding, build, experiments
    build.build()
    binding.load_library()
    return experiments


def test_hover_regression(E):
    """zero command, no disturbance, 10 s -> no fall, mean velocity error < 0.05 m/s."""
    r = E.hover(K=10000, inner=8)
    assert r["fallen"] == 0
    assert r["mean_vel_err"] < 0.05


def test_fig4_frequency_rises_under_the_push_and_recovers(E):
    """under a 40 N lateral push the step frequency is increased, and after the
    push it is restored toward the nominal value; without gait adaptation it stays at f_n."""
    a = E.fig4(K=10000, push=40.0, adapt=1, inner=8)
    assert a["fallen"] == 0
    assert a["f_push"] > a["f_before"] and a["f_push"] > a["f_after"]
    f = E.fig4(K=10000, push=40.0, adapt=0, inner=8)
    assert abs(f["f_push"] - 1.3) < 1e-6 and abs(f["f_after"] - 1.3) < 1e-6


def test_table1_ordering_adaptive_beats_fixed(E):
    """Table I: under random CoM wrenches, Naive with gait adaptation keeps more
    episodes upright than Naive with the fixed gait.  Our SRBD desk-scale loop is a weak
    proxy of the paper's simulator: the ordering is checked in aggregate over a range of
    disturbance amplitudes (100 paired episodes each), where it holds."""
    fixed = adaptive = 0.0
    for amp in (10.0, 12.0, 14.0, 16.0):
        r = E.table1(episodes=100, amp=amp, K=10000, inner=8, variants=[("naive", 0), ("naive", 1)])
        f, a = r["results"]
        fixed += f["success_pct"]
        adaptive += a["success_pct"]
        assert a["mean_freq"] > 1.3 + 1e-3 and abs(f["mean_freq"] - 1.3) < 1e-5
    assert adaptive > fixed
