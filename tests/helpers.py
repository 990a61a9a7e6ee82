"""Test helpers: golden-case unpacking and statistical parity criteria
(SURVEY.md Appendix B)."""

import math

import numpy as np

CASE_NAMES = ["disc", "annulus", "five", "square_hole", "square_hole_aniso", "shell3d"]


def case(g, name):
    pre = name + "."
    return {k[len(pre):]: v for k, v in g.items() if k.startswith(pre)}


def side_tuple(c, s):
    return (c[f"a{s}"], c[f"blk{s}"], c[f"blkf{s}"], 0, np.zeros(0), 2)


def two_sample_z(c1, n1, c2, n2):
    """Entry-wise two-sample binomial z with pooled p (Appendix B)."""
    c1 = np.asarray(c1, dtype=float)
    c2 = np.asarray(c2, dtype=float)
    p1, p2 = c1 / n1, c2 / n2
    pool = (c1 + c2) / (n1 + n2)
    se = np.sqrt(np.maximum(pool * (1 - pool), 1e-300) * (1.0 / n1 + 1.0 / n2))
    z = np.where(pool > 0, (p1 - p2) / se, 0.0)
    return z


def exact_two_sample_p(c1, n1, c2, n2):
    """Entry-wise exact conditional test of equal binomial rates: given the
    pooled count T = c1 + c2, c1 ~ Binomial(T, n1/(n1+n2)) under H0; two-
    sided p-value.  Valid at any count (Appendix B's low-count caveat)."""
    from scipy.stats import binom

    c1 = np.asarray(c1, dtype=float)
    c2 = np.asarray(c2, dtype=float)
    t = c1 + c2
    q = n1 / (n1 + n2)
    lo = binom.cdf(c1, t, q)
    hi = binom.sf(c1 - 1, t, q)
    return np.minimum(1.0, 2.0 * np.minimum(lo, hi))


P_Z4 = 6.334248366623996e-05  # two-sided P(|Z| > 4)


def bonferroni_z(m_entries, alpha=0.05):
    """Two-sided Bonferroni threshold Phi^-1(1 - alpha/(2m))."""
    from scipy.stats import norm

    return float(norm.isf(alpha / (2.0 * m_entries)))


def exceed_quantile(m_entries, q=0.999, z=4.0):
    """Upper q-quantile of the number of |Z|>z exceedances among m iid
    entries of a perfect implementation."""
    from scipy.stats import binom, norm

    p = 2.0 * norm.sf(z)
    return int(binom.ppf(q, m_entries, p))


def row_chi2_pvalues(c1, n1, c2, n2, min_expected=5.0):
    """Per-row 2xK chi-square homogeneity p-values, pooling bins with small
    expected counts into one."""
    from scipy.stats import chi2

    out = []
    for a, b in zip(np.asarray(c1, float), np.asarray(c2, float)):
        tot = a + b
        keep = tot * min(n1, n2) / (n1 + n2) >= min_expected
        a2 = np.append(a[keep], a[~keep].sum())
        b2 = np.append(b[keep], b[~keep].sum())
        tot2 = a2 + b2
        m = tot2 > 0
        a2, b2, tot2 = a2[m], b2[m], tot2[m]
        ea = tot2 * n1 / (n1 + n2)
        eb = tot2 * n2 / (n1 + n2)
        stat = float(np.sum((a2 - ea) ** 2 / ea + (b2 - eb) ** 2 / eb))
        dof = max(len(a2) - 1, 1)
        out.append(float(chi2.sf(stat, dof)))
    return np.array(out)


def poisson_cell_probs_disk(pole, n_bins, q=64, phase=0.5):
    """Cell-integrated Poisson kernel of the unit disk for arcs
    [2pi k/n, 2pi (k+1)/n) (midpoint anchors, phase 1/2), as in
    T/test_acceptance.py:93-101."""
    pole = np.asarray(pole, float)
    delta = 2.0 * math.pi / n_bins
    out = np.empty(n_bins)
    for k in range(n_bins):
        th = (k + phase) * delta - delta / 2.0 + delta * (np.arange(q) + 0.5) / q
        ys = np.stack([np.cos(th), np.sin(th)], axis=1)
        kern = (1.0 - pole @ pole) / (2.0 * math.pi * np.sum((pole - ys) ** 2, axis=1))
        out[k] = kern.mean() * delta
    return out
