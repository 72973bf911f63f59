"""Band-mask lowering edge cases (plan._band_from_cond): strict bounds with non-integer constants
keep the reference's set, and masks the kernels cannot express raise instead of silently running
unmasked (a window <= 0 reads as 'no window' in every kernel)."""
import math

import numpy as np
import pytest

from paper_2502_15349_b200 import hooklang as H, plan as P
from paper_2502_15349_b200.errors import UnsupportedError


def band_of(expr: str) -> P.Band:
    b = P.Band()
    fn = type("F", (), {"expr": H.parse(expr), "source": expr})()
    assert P._mask_kind(fn, {}, b) is not None, expr
    return b


@pytest.mark.parametrize("expr", [
    "where(qidx - kidx < 2.5, s, -inf)", "where(qidx - kidx <= 2.5, s, -inf)",
    "where(kidx < qidx + 0.5, s, -inf)", "where(kidx <= qidx, s, -inf)",
    "where(qidx - kidx < 4, s, -inf)", "where(kidx - qidx <= -1, s, -inf)",
    "where(2 * kidx < 2 * qidx + 3, s, -inf)", "s * where(qidx - kidx < 7, 1, 0)"])
def test_band_keeps_exactly_the_reference_set(expr):
    b = band_of(expr)
    i = np.arange(40)[:, None].astype(float)
    j = np.arange(40)[None, :].astype(float)
    cond = H.parse(expr).args[0] if isinstance(H.parse(expr), H.Fn) else \
        H.parse(expr).rhs.args[0]
    env = {"qidx": i, "kidx": j}

    def ev(n):
        if isinstance(n, H.Name):
            return env[n.name]
        if isinstance(n, H.Num):
            return n.value
        a, c = ev(n.lhs), ev(n.rhs)
        return {"+": a + c, "-": a - c, "*": a * c, "<": a < c, "<=": a <= c, ">": a > c,
                ">=": a >= c}[n.op]
    want = np.broadcast_to(ev(cond), (40, 40))
    assert np.array_equal(b.keep(i.astype(int), j.astype(int)), want), (expr, b)


def test_lower_key_bound_at_the_diagonal_is_unsupported():
    b = band_of("where(kidx > qidx, s, -inf)")
    with pytest.raises(UnsupportedError):
        _ = b.kernel_window


def test_window_of_a_strict_noninteger_bound():
    assert band_of("where(qidx - kidx < 2.5, s, -inf)").window == 3
    assert not math.isnan(band_of("where(qidx - kidx < 4, s, -inf)").kernel_window)
