// gate.h -- host-side power-law check of Alg. 2 line 3.
#pragma once
#include <cstdint>
#include <vector>

namespace cc {
namespace gate {

struct LsFit {
  double alpha = 0, r2 = 0;
  uint64_t dmax = 0;
  int bins = 0;
  bool scale_free = false;
};
struct KsFit {
  double ks = 0, alpha = 0;
  uint32_t xmin = 0;
  bool valid = false;
};

// Degree distribution as sparse (degree, count) pairs with degree >= 1, ascending.
using Hist = std::vector<std::pair<uint64_t, uint64_t>>;

// Gate G: least squares of log10 density on log10 bin centre over
// log bins floor(10^(k/5)); scale-free iff dmax >= 100, R^2 >= 0.7, 1 < alpha < 3.5.
LsFit fit_ls(const Hist& h);
// Paper's statistic: discrete power law (Clauset et al.), approximate MLE, K-S distance
// at the support points, x_min minimising it over admissible candidates.
KsFit fit_ks(const Hist& h);
double hurwitz_zeta(double s, double q);

}  // namespace gate
}  // namespace cc
