"""Pin of the aliased collocation variant (DESIGN.md §6 P24): the padded fast
algorithm with a product grid of P < 3N/2 − 2 points (P = N: the classical collocation spectral method) must
equal the brute-force double sum over pairs with l + m ≡ k (mod P), and differ from the exact Galerkin sum."""
import numpy as np
import pytest

from oracle import fks_oracle as o

L = 13.242640687119286


@pytest.mark.parametrize("N", [4, 6, 8, 12])
@pytest.mark.parametrize("kernel", [0, 1])
def test_P24_aliased_fast_equals_aliased_direct_sum(N, kernel):
    tb = o.build_tables(N, L, M=16, M_r=4, kernel=kernel)
    rng = np.random.default_rng(24 + N + 100 * kernel)
    f = rng.random((N, N, N)) - (0.3 if kernel else 0.0)
    exact = o.collision_direct(f, tb)
    for P in sorted({N, N + 1, N + 2, 3 * N // 2 - 3}):
        if P < N:
            continue
        fast = o.collision_fast(f, tb, P)
        direct = o.collision_direct(f, tb, P=P)
        assert np.abs(fast - direct).max() <= 1e-12 * np.abs(direct).max(), P
        if P <= 3 * N // 2 - 3:  # pairs with l + m = k -+ P exist: a different operator
            assert np.abs(direct - exact).max() > 1e-6 * np.abs(exact).max(), P
        else:  # no pair wraps onto K' any more (A10): the exact Galerkin sum
            assert np.abs(direct - exact).max() <= 1e-12 * np.abs(exact).max(), P
    # P >= 3N/2 - 2: no aliasing left, the exact Galerkin sum
    assert np.abs(o.collision_direct(f, tb, P=3 * N // 2 - 2) - exact).max() <= 1e-14 * np.abs(exact).max()
