"""Host logic of the adaptive incrementation (paper_2103_04770_b200.run.adaptive_schedule, A-34)
against a mock increment solver (CPU only)."""
import pytest

from paper_2103_04770_b200.run import adaptive_schedule


def test_fixed_steps_when_every_increment_converges():
    acc, cuts, ok = adaptive_schedule(lambda E: True, 0.01, 1e-3)
    assert ok and cuts == 0 and len(acc) == 10
    assert acc[-1] == pytest.approx(0.01, abs=1e-15)


def test_cutback_and_regrowth():
    # increments larger than 2.6e-4 fail beyond E = 0.004 (a "softening" region)
    last = [0.0]

    def solve(E):
        ok = E <= 0.004 + 1e-15 or E - last[0] <= 2.6e-4
        if ok:
            last[0] = E
        return ok

    acc, cuts, ok = adaptive_schedule(solve, 0.006, 1e-3, grow=1.5, grow_after=2)
    assert ok and acc[-1] == pytest.approx(0.006)
    assert cuts >= 2
    steps = [b - a for a, b in zip([0.0] + acc[:-1], acc)]
    assert max(steps[acc.index(min(a for a in acc if a > 0.004)):]) <= 2.6e-4 + 1e-15
    assert all(b > a for a, b in zip(acc, acc[1:]))          # monotone loading


def test_gives_up_below_min_step():
    acc, cuts, ok = adaptive_schedule(lambda E: E < 0.002, 0.01, 1e-3, dE_min=1e-5)
    assert not ok and acc[-1] < 0.002
    # every failure halves: reaching 1e-5 from 1e-3 takes at most log2(100) + 1 cuts per stall
    assert cuts <= 8 * 2


def test_doubling_schedule_and_early_stop():
    """grow = 2 (the golden curves' rule: halve on failure, x2 after two first-try successes, never
    beyond dE) keeps every accepted target a dyadic multiple of dE, and stop() ends the run after
    the accepted increment that triggers it."""
    last = [0.0]

    def solve(E):
        ok = E - last[0] <= 2.5e-4 + 1e-15 or E <= 0.002 + 1e-15
        if ok:
            last[0] = E
        return ok

    acc, cuts, ok = adaptive_schedule(solve, 0.004, 1e-3, grow=2.0, stop=lambda: last[0] >= 0.003 - 1e-15)
    assert ok and cuts >= 2
    assert acc[-1] == pytest.approx(0.003, abs=1e-15)          # stopped, not run to 0.004
    for E in acc:
        q = E / 2.5e-4
        assert abs(q - round(q)) < 1e-9                           # dyadic targets
