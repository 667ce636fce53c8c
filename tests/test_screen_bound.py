"""The SYRK engine's mode-3 K2 screen (engine.cu k2_screen_scaled<true>,
E3_SCREEN_V2) against exact K2 scores, emulated on the CPU in fp32.

The device returns ln2 * sum_c (m_c + 1/2) lg2(m_c) - sum_c (G[r0_c] + G[r1_c])
(m = r0 + r1 + 1, G[n] = fl32(ln n! - alpha n)) and passes a triple when that
is <= threshold + kshift_st, kshift_st = (1 + alpha) N + 27 - 13.5 ln(2 pi) +
k2_screen_margin_st (engine.cu). A triple in the top-k has score <= threshold,
so the screen must never exceed score + kshift_st: checked here for random and
adversarial (skewed, zero-heavy) cell tables with lg2 perturbed by the
assumed approximation error in the worst direction, in the device's f32x2
lane order. The margin is restated from engine.cu (test infrastructure).
"""
import math

import numpy as np
import pytest

U = 2.0 ** -24
E = 2.0 ** -20
LN2 = math.log(2.0)
LN2_F = np.float32(LN2)


def margin_st(gmax, n):
    """engine.cu k2_screen_margin_st."""
    a = (n + 41.0) * math.log2(n + 2.0)
    gp = 54.0 * gmax
    smax = n * LN2 + 27.0 * math.log(n + 1.0) + 1.0
    err = LN2 * E * (n + 41.0) + 13.0 * U * LN2 * a + 56.0 * U * gmax + 12.0 * U * gp
    return 2.0 * err * (1.0 + 8.0 * U) + 1e-9 * smax + 1e-6


def f32(x):
    return np.float32(x)


def fma32(a, b, c):
    # a*b is exact in float64 for float32 inputs; one rounding to float32
    return np.float32(np.float64(a) * np.float64(b) + np.float64(c))


def tables(n):
    alpha = math.log(n + 1.0) - 1.2785
    lf = np.array([math.lgamma(k + 1.0) for k in range(n + 2)])
    g = lf - alpha * np.arange(n + 2)
    return alpha, lf, g.astype(np.float32), float(np.max(np.abs(g)))


def screen_v2(r0, r1, gt, lg_sign):
    """Device order: cells 0..25 in pairs into lanes (as[(c>>1)&1], lo/hi),
    the last cell separately; FFMA for the pooled term, adds for the table."""
    as_ = [[f32(0), f32(0)], [f32(0), f32(0)]]
    ag = [[f32(0), f32(0)], [f32(0), f32(0)]]
    def lg2(m):
        return f32(math.log2(m) + lg_sign * E)
    for c in range(0, 26, 2):
        k = (c >> 1) & 1
        for e in range(2):
            m = f32(r0[c + e] + r1[c + e] + 1)
            mh = f32(r0[c + e] + r1[c + e] + 1.5)
            as_[k][e] = fma32(mh, lg2(float(m)), as_[k][e])
        for e in range(2):
            pair = f32(gt[r0[c + e]] + gt[r1[c + e]])
            ag[k][e] = f32(ag[k][e] + pair)
    m = f32(r0[26] + r1[26] + 1)
    s_last = f32(f32(m + f32(0.5)) * lg2(float(m)))
    g_last = f32(gt[r0[26]] + gt[r1[26]])
    s = f32(f32(f32(as_[0][0] + as_[1][0]) + f32(as_[0][1] + as_[1][1])) + s_last)
    g = f32(f32(f32(ag[0][0] + ag[1][0]) + f32(ag[0][1] + ag[1][1])) + g_last)
    return fma32(s, LN2_F, -g)


def k2_exact(r0, r1, lf):
    return float(sum(lf[a + b + 1] - lf[a] - lf[b] for a, b in zip(r0, r1)))


def draws(rng, n0, n1, count):
    for t in range(count):
        kind = t % 4
        if kind == 0:    # balanced cells
            p0 = p1 = rng.dirichlet(np.ones(27) * 5)
        elif kind == 1:  # skewed: a few large cells, many tiny / empty ones
            p0 = rng.dirichlet(np.ones(27) * 0.2)
            p1 = rng.dirichlet(np.ones(27) * 0.2)
        elif kind == 2:  # maf-0.3-like genotype products, strong class effect
            g = np.array([0.49, 0.42, 0.09])
            base = np.einsum("i,j,k->ijk", g, g, g).ravel()
            p0 = base
            p1 = rng.dirichlet(base * 50)
        else:            # everything in one cell
            p0 = np.eye(27)[rng.integers(27)]
            p1 = np.eye(27)[rng.integers(27)]
        yield rng.multinomial(n0, p0), rng.multinomial(n1, p1)


@pytest.mark.parametrize("n0,n1", [(2048, 2048), (8192, 8192), (16383, 16383), (3000, 9000)])
def test_screen_never_exceeds_score_plus_shift(n0, n1):
    n = n0 + n1
    alpha, lf, gt, gmax = tables(n)
    shift = (1.0 + alpha) * n + 27.0 - 13.5 * math.log(2.0 * math.pi)
    marg = margin_st(gmax, n)
    rng = np.random.default_rng(n0 * 7 + n1)
    worst = -math.inf
    for r0, r1 in draws(rng, n0, n1, 40):
        score = k2_exact(r0, r1, lf)
        for sign in (1.0, -1.0):
            sc = float(screen_v2(r0, r1, gt, sign))
            # pass condition on the device: sc <= thr + shift + margin; a
            # top-k triple has score <= thr, so sc - shift - margin <= score
            slack = sc - shift - score
            worst = max(worst, slack)
            assert slack <= marg, (slack, marg)
    # the bound is not vacuous: the screen tracks the score closely
    assert worst > -2.0, worst
    assert marg < 1.5


def test_margin_matches_design_numbers():
    _, _, _, gmax = tables(16384)
    assert 0.5 < margin_st(gmax, 16384) < 0.8  # 0.65 nats at N = 16384
