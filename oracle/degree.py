"""Graph-structure prediction of Alg. 2.  TEST INFRASTRUCTURE.

* :func:`degree_distribution` -- Alg. 2 line 2: "each undirected edge
  (u,v) [is stored] as two directed edges ... We compute the degree distribution D of the
  graph by doing a global sort of edge list by the source vertex. Through a linear scan
  over the sorted edge list, we compute the degree of each vertex".
  Degree = number of arcs with that source, multiplicity counted; a self-loop {x,x}
  gives two arcs (x,x), hence degree 2.  D[d] = #vertices of degree d,
  d >= 1 (C10).  Written as the paper says: sort arcs by source, run lengths, count.
* :func:`gate_ls` -- gate G (north star "degree histogram plus log-log
  least-squares fit"): log-binned density, ordinary least squares in log10-log10.
* :func:`ks_powerlaw` -- the paper's statistic ("the statistical framework
  described by Clauset et al. to fit a power-law curve to the discrete graph degree
  distribution, and estimate the goodness of fit with one-sample Kolmogorov-Smirnov
  (K-S) test"; threshold tau = 0.05): discrete power law with the
  approximate MLE alpha = 1 + N / sum ln(d / (x_min - 1/2)), model CDF from the Hurwitz
  zeta function, x_min chosen to minimise the K-S distance (readings R8-R9).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import zeta as hurwitz_zeta

# gate G constants (reading R7)
BINS_PER_DECADE = 5
GATE_MIN_DMAX = 100
GATE_MIN_R2 = 0.7
GATE_ALPHA_LO = 1.0
GATE_ALPHA_HI = 3.5
KS_XMIN_CAP = 200
KS_XMIN_FACTOR = 10
KS_TAU = 0.05


def degree_distribution(n, edges):
    """Returns (deg[n], D) with D a dict-like array hist[d] for d in [0, d_max]."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    # arcs (u,v) and (v,u) for every undirected edge
    src = np.concatenate([e[:, 0], e[:, 1]])
    src_sorted = np.sort(src, kind="stable")            # "global sort ... by the source"
    deg = np.zeros(n, dtype=np.int64)
    if src_sorted.shape[0]:
        head = np.empty(src_sorted.shape[0], bool)
        head[0] = True
        head[1:] = src_sorted[1:] != src_sorted[:-1]
        starts = np.flatnonzero(head)
        runs = np.diff(np.append(starts, src_sorted.shape[0]))   # "linear scan" run lengths
        deg[src_sorted[starts]] = runs
    dmax = int(deg.max()) if n else 0
    hist = np.bincount(deg, minlength=dmax + 1).astype(np.int64)
    hist[0] = 0  # degree-0 ids are not part of D (C10)
    return deg, hist


def log_bin_edges(dmax):
    """Bin edges floor(10^(k/5)) de-duplicated, closed by dmax+1 (C11)."""
    edges = []
    k = 0
    while True:
        e = int(math.floor(10.0 ** (k / BINS_PER_DECADE) * (1.0 + 1e-12)))
        if e > dmax:
            break
        if not edges or edges[-1] != e:
            edges.append(e)
        k += 1
    edges.append(dmax + 1)
    return edges


def gate_ls(hist):
    """Gate G: returns dict(alpha, r2, dmax, bins, scale_free)."""
    hist = np.asarray(hist, dtype=np.int64)
    nz = np.flatnonzero(hist)
    nz = nz[nz >= 1]
    if nz.shape[0] == 0:
        return dict(alpha=float("nan"), r2=float("nan"), dmax=0, bins=0, scale_free=False)
    dmax = int(nz[-1])
    N = float(hist[1:].sum())
    be = log_bin_edges(dmax)
    cum = np.concatenate([[0], np.cumsum(hist)])  # cum[d] = sum hist[0..d-1]
    xs, ys = [], []
    for lo, hi in zip(be[:-1], be[1:]):
        cnt = float(cum[hi] - cum[lo])               # degrees in [lo, hi)
        if cnt <= 0:
            continue
        width = hi - lo
        density = cnt / (N * width)
        centre = math.sqrt(lo * (hi - 1))
        xs.append(math.log10(centre))
        ys.append(math.log10(density))
    k = len(xs)
    if k < 3:
        return dict(alpha=float("nan"), r2=float("nan"), dmax=dmax, bins=k, scale_free=False)
    x = np.asarray(xs)
    y = np.asarray(ys)
    xm, ym = x.mean(), y.mean()
    sxx = float(((x - xm) ** 2).sum())
    sxy = float(((x - xm) * (y - ym)).sum())
    syy = float(((y - ym) ** 2).sum())
    slope = sxy / sxx
    r2 = (sxy * sxy) / (sxx * syy) if syy > 0 else 1.0
    alpha = -slope
    sf = (dmax >= GATE_MIN_DMAX) and (r2 >= GATE_MIN_R2) and (GATE_ALPHA_LO < alpha < GATE_ALPHA_HI)
    return dict(alpha=alpha, r2=r2, dmax=dmax, bins=k, scale_free=bool(sf))


def ks_powerlaw(hist):
    """Clauset-style discrete fit; returns dict(ks, alpha, xmin) (ks = nan if no admissible
    x_min).  Candidates: distinct degrees x_min >= 1 with d_max >= 10 x_min and
    x_min <= 200.  K-S distance evaluated at the support points
    (distinct degrees >= x_min): D = max |S(x) - P(x)|, S the empirical CDF of the tail,
    P(x) = 1 - zeta(alpha, x+1) / zeta(alpha, x_min)."""
    hist = np.asarray(hist, dtype=np.int64)
    ds = np.flatnonzero(hist)
    ds = ds[ds >= 1]
    best = dict(ks=float("nan"), alpha=float("nan"), xmin=0)
    if ds.shape[0] == 0:
        return best
    dmax = int(ds[-1])
    cnt = hist[ds].astype(np.float64)
    for j, xmin in enumerate(ds):
        xmin = int(xmin)
        if KS_XMIN_FACTOR * xmin > dmax or xmin > KS_XMIN_CAP:
            continue
        td = ds[j:].astype(np.float64)
        tc = cnt[j:]
        ntail = tc.sum()
        alpha = 1.0 + ntail / float((tc * np.log(td / (xmin - 0.5))).sum())
        S = np.cumsum(tc) / ntail
        P = 1.0 - hurwitz_zeta(alpha, td + 1.0) / hurwitz_zeta(alpha, float(xmin))
        D = float(np.max(np.abs(S - P)))
        if not (D >= best["ks"]):  # strict improvement (nan-safe): smallest x_min wins ties
            best = dict(ks=D, alpha=float(alpha), xmin=xmin)
    return best
