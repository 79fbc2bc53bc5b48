"""Host logic of the NEXT-1 break-even sweep: crossing density by linear
interpolation between bracketing sweep points (closed-form cases)."""
import pytest

from paper_2005_04091_b200.breakeven import break_even_density


def test_linear_crossing_midpoint():
    # sparse time grows linearly 1..5 over densities .1...5; dense = 3 -> crossing at .3
    assert break_even_density([0.1, 0.2, 0.3, 0.4, 0.5], [1, 2, 3, 4, 5], 3.0) == pytest.approx(0.3)
    assert break_even_density([0.1, 0.5], [1.0, 5.0], 2.0) == pytest.approx(0.2)


def test_never_and_always():
    assert break_even_density([0.1, 0.5, 1.0], [1, 2, 3], 10.0) is None
    assert break_even_density([0.1, 0.5, 1.0], [5, 6, 7], 1.0) == 0.1


def test_validation():
    with pytest.raises(ValueError):
        break_even_density([0.2, 0.1], [1, 2], 1.0)
    with pytest.raises(ValueError):
        break_even_density([], [], 1.0)
