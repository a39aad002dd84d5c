// gate.cpp -- power-law check of the degree distribution (host, FP64).
//
// The paper classifies a graph as scale-free when the one-sample K-S statistic of a
// discrete power-law fit (Clauset et al.) to its degree distribution is below a user
// threshold tau (Alg. 2 line 3 PAPER.md:258, tau = 0.05 PAPER.md:345).
// SURVEY.md §0.3 / C11 measured that this statistic does not separate the synthetic
// configs here, so the default decision is gate G, the north star's "degree histogram
// plus log-log least-squares fit"; the K-S statistic is still computed (for the report,
// and for the decision under CC_FLAG_GATE_KS).  Constants: DESIGN.md §2 readings R7-R9.
#include "gate.h"

#include <cmath>
#include <limits>

namespace cc {
namespace gate {

static const int kBinsPerDecade = 5;
static const uint64_t kMinDmax = 100;
static const double kMinR2 = 0.7, kAlphaLo = 1.0, kAlphaHi = 3.5;
static const uint64_t kXminCap = 200, kXminFactor = 10;

LsFit fit_ls(const Hist& h) {
  LsFit f;
  if (h.empty()) return f;
  f.dmax = h.back().first;
  double N = 0;
  for (auto& e : h) N += (double)e.second;
  // bin edges floor(10^(k/5)), de-duplicated, closed by dmax+1
  std::vector<uint64_t> edges;
  for (int k = 0;; k++) {
    uint64_t e = (uint64_t)std::floor(std::pow(10.0, (double)k / kBinsPerDecade) * (1.0 + 1e-12));
    if (e > f.dmax) break;
    if (edges.empty() || edges.back() != e) edges.push_back(e);
  }
  edges.push_back(f.dmax + 1);
  std::vector<double> xs, ys;
  size_t j = 0;
  for (size_t b = 0; b + 1 < edges.size(); b++) {
    uint64_t lo = edges[b], hi = edges[b + 1];
    double cnt = 0;
    while (j < h.size() && h[j].first < lo) j++;
    size_t jj = j;
    while (jj < h.size() && h[jj].first < hi) cnt += (double)h[jj++].second;
    j = jj;
    if (cnt <= 0) continue;
    double density = cnt / (N * (double)(hi - lo));
    double centre = std::sqrt((double)lo * (double)(hi - 1));
    xs.push_back(std::log10(centre));
    ys.push_back(std::log10(density));
  }
  f.bins = (int)xs.size();
  if (f.bins < 3) {
    f.alpha = f.r2 = std::numeric_limits<double>::quiet_NaN();
    return f;
  }
  double xm = 0, ym = 0;
  for (int i = 0; i < f.bins; i++) { xm += xs[i]; ym += ys[i]; }
  xm /= f.bins; ym /= f.bins;
  double sxx = 0, sxy = 0, syy = 0;
  for (int i = 0; i < f.bins; i++) {
    double dx = xs[i] - xm, dy = ys[i] - ym;
    sxx += dx * dx; sxy += dx * dy; syy += dy * dy;
  }
  double slope = sxy / sxx;
  f.r2 = syy > 0 ? (sxy * sxy) / (sxx * syy) : 1.0;
  f.alpha = -slope;
  f.scale_free = f.dmax >= kMinDmax && f.r2 >= kMinR2 && f.alpha > kAlphaLo && f.alpha < kAlphaHi;
  return f;
}

// Hurwitz zeta(s, q) = sum_{k>=0} (q+k)^-s, s > 1, q > 0, by Euler-Maclaurin summation:
// N direct terms, the integral tail, and Bernoulli corrections.
double hurwitz_zeta(double s, double q) {
  const int N = 16;
  double sum = 0;
  for (int k = 0; k < N; k++) sum += std::pow(q + k, -s);
  double a = q + N;
  double tail = std::pow(a, 1.0 - s) / (s - 1.0) + 0.5 * std::pow(a, -s);
  // B_{2j}/(2j)!
  static const double B[] = {1.0 / 6.0,        -1.0 / 30.0,         1.0 / 42.0,
                             -1.0 / 30.0,      5.0 / 66.0,          -691.0 / 2730.0,
                             7.0 / 6.0,        -3617.0 / 510.0};
  double fact = 1.0;      // (2j)!
  double poch = s;        // s (s+1) ... (s+2j-2)
  double apow = std::pow(a, -s - 1.0);
  for (int j = 1; j <= 8; j++) {
    fact *= (double)(2 * j - 1) * (double)(2 * j);
    tail += B[j - 1] / fact * poch * apow;
    poch *= (s + 2 * j - 1) * (s + 2 * j);
    apow /= a * a;
  }
  return sum + tail;
}

KsFit fit_ks(const Hist& h) {
  KsFit best;
  best.ks = std::numeric_limits<double>::quiet_NaN();
  if (h.empty()) return best;
  const uint64_t dmax = h.back().first;
  const size_t K = h.size();
  for (size_t j = 0; j < K; j++) {
    const uint64_t xmin = h[j].first;
    if (kXminFactor * xmin > dmax || xmin > kXminCap) continue;
    double ntail = 0, slog = 0;
    for (size_t t = j; t < K; t++) {
      ntail += (double)h[t].second;
      slog += (double)h[t].second * std::log((double)h[t].first / ((double)xmin - 0.5));
    }
    const double alpha = 1.0 + ntail / slog;
    const double zmin = hurwitz_zeta(alpha, (double)xmin);
    double cum = 0, D = 0;
    for (size_t t = j; t < K; t++) {
      cum += (double)h[t].second;
      double S = cum / ntail;
      double P = 1.0 - hurwitz_zeta(alpha, (double)h[t].first + 1.0) / zmin;
      double dd = std::fabs(S - P);
      if (dd > D) D = dd;
    }
    if (!best.valid || D < best.ks) {
      best.ks = D; best.alpha = alpha; best.xmin = (uint32_t)xmin; best.valid = true;
    }
  }
  return best;
}

}  // namespace gate
}  // namespace cc
