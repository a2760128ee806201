"""The lazy oracle (on-demand, memoised evaluation of §3.2) equals the eager oracle pair by pair
(same formulas, same row order inside Z; only the evaluation order differs)."""
import numpy as np
import pytest

from oracle.lazy import LazyRecompression

from conftest import oracle_run


@pytest.mark.parametrize("name", ["P1", "P3"])
def test_lazy_equals_eager(name):
    rc = oracle_run(name)
    lz = LazyRecompression(rc.st, rc.eps)
    for l in rc.st.active_levels:
        for (t, c) in rc.st.basis_pairs[l][::3]:
            assert np.array_equal(lz.R(t, c), rc.R[(t, c)])
    for side in ("row", "col"):
        res = getattr(rc, side)
        for key in list(res.sigma)[::2]:
            tr = lz.truncate(side, *key)
            assert np.array_equal(lz.Zhat(side, *key), res.Zhat[key])
            assert tr["rank"] == res.rank[key]
            assert np.array_equal(tr["sigma"], res.sigma[key])
            assert np.array_equal(tr["C"], res.C[key])
