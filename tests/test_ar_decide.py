"""The autoregressive decision shortcut of zxs_dedup.cuh (`ar_decide`): a float
quotient with a 4e-7 relative margin decides `!(u < clamp(cur / prev))` and the
ratio-error check exactly whenever it answers; otherwise the IEEE quotient is
used. Restated with numpy float32 (IEEE round-to-nearest division is at least
as accurate as __fdividef's 2-ulp bound the margin covers) and checked against
the reference's double-precision rule (sampler.cpp:84-99) on adversarial
inputs: uniforms placed at, and within a few ulps of, the exact ratios."""
import numpy as np


def exact(cur, prev, u):
    with np.errstate(all="ignore"):
        ratio = np.float64(cur) / np.float64(prev)
    err = not (ratio > -1e-6 and ratio < 1.0 + 1e-6)
    cl = ratio if 0.0 < ratio else 0.0
    cl = cl if cl < 1.0 else 1.0
    return (not (u < cl)), err


def shortcut(cur, prev, u, skew=0):
    """The device rule with its float quotient moved `skew` float ulps off the
    correctly rounded one (__fdividef is within 2 ulps)."""
    ac, ap = abs(cur), abs(prev)
    if 1e-30 < ap < 1e30 and (ac == 0.0 or 1e-30 < ac < 1e30):
        with np.errstate(all="ignore"):
            qf = np.float32(cur) / np.float32(prev)
            for _ in range(abs(skew)):
                qf = np.nextafter(qf, np.float32(np.inf if skew > 0 else -np.inf))
        q = float(qf)
        d = 4e-7 * abs(q) + 1e-37
        if q - d > -1e-6 and q + d < 1.0 + 1e-6:
            if u < q - d:
                return False, False
            if u > q + d:
                return True, False
    return exact(cur, prev, u)


def test_shortcut_matches_exact_rule():
    rng = np.random.default_rng(11)
    n = 0
    for _ in range(20000):
        prev = float(rng.uniform(1e-3, 1e4)) * (1 if rng.random() < 0.95 else -1)
        kind = rng.integers(0, 5)
        if kind == 0:
            cur = prev  # ratio exactly 1
        elif kind == 1:
            cur = 0.0
        elif kind == 2:
            cur = prev * float(rng.uniform(-1e-5, 1e-5))  # near the lower error bound
        elif kind == 3:
            cur = prev * (1.0 + float(rng.uniform(-3e-6, 3e-6)))  # near the upper error bound
        else:
            cur = prev * float(rng.random())
        ratio = np.float64(cur) / np.float64(prev)
        base = min(max(float(ratio), 0.0), np.nextafter(1.0, 0.0))
        us = [base, np.nextafter(base, 0.0), np.nextafter(base, 1.0), float(rng.random()),
              base * (1 + 3e-7), base * (1 - 3e-7), 0.0]
        for u in us:
            u = min(max(float(u), 0.0), np.nextafter(1.0, 0.0))
            u = np.floor(u * 2.0 ** 53) / 2.0 ** 53  # uniform_at values are multiples of 2^-53
            want = exact(cur, prev, u)
            for skew in (-2, -1, 0, 1, 2):
                assert shortcut(cur, prev, u, skew) == want, (cur, prev, u, skew)
            n += 1
    assert n > 100000
