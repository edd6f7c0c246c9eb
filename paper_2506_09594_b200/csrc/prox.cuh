// Scalar proximity operators of the seven tenrec penalties, evaluated in fp64.
//
// Mirrors tenrec/penalties.py (file:line per family below).  Encoding
// (kind, p0, p1) is the C-ABI's: 0 l1, 1 firm(gamma), 2 mcp(gamma),
// 3 scad(a), 4 lq(q), 5 capped-lq(q, theta), 6 log(gamma).
#pragma once

#include <math.h>

namespace tr {

struct Penalty {
  int kind;
  double p0, p1;
};

__host__ __device__ inline double pen_value(const Penalty& p, double t, double mu) {
  switch (p.kind) {
    case 0:  // penalties.py:71-72
      return mu * t;
    case 1:
    case 2: {  // penalties.py:83-87
      double g = p.p0;
      return t <= g * mu ? mu * t - t * t / (2.0 * g) : g * mu * mu / 2.0;
    }
    case 3: {  // penalties.py:127-133
      double a = p.p0;
      if (t <= mu) return mu * t;
      if (t <= a * mu) return (2.0 * a * mu * t - t * t - mu * mu) / (2.0 * (a - 1.0));
      return mu * mu * (a + 1.0) / 2.0;
    }
    case 4:  // penalties.py:161-162
      return mu * pow(t, p.p0);
    case 5:  // penalties.py:228-229
      return mu * pow(fmin(t, p.p1), p.p0);
    default:  // penalties.py:259-260
      return mu * log1p(t / p.p0);
  }
}

// Lq prox on a magnitude (penalties.py:164-206).  The reference iterates Newton
// jointly over an array and stops on the array-wide max step; per element the
// iterates are identical until convergence and later steps are below 1e-12.
__host__ __device__ inline double lq_prox_abs(double q, double mu, double a) {
  if (q == 1.0) return fmax(a - mu, 0.0);
  double xh = pow(2.0 * mu * (1.0 - q), 1.0 / (2.0 - q));
  double thr = xh + mu * q * pow(xh, q - 1.0);
  if (!(a > thr)) return 0.0;
  double x = a;
  for (int it = 0; it < 50; ++it) {
    double g = x + mu * q * pow(x, q - 1.0) - a;
    double dg = 1.0 + mu * q * (q - 1.0) * pow(x, q - 2.0);
    double step = g / dg;
    x = fmax(x - step, 1e-300);
    if (fabs(step) < 1e-12) return x;
  }
  double lo = xh, hi = a;  // bisection fallback
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    if (mid + mu * q * pow(mid, q - 1.0) - a < 0) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

__host__ __device__ inline double prox_abs(const Penalty& p, double mu, double a) {
  switch (p.kind) {
    case 0:  // penalties.py:74-75
      return fmax(a - mu, 0.0);
    case 1:
    case 2: {  // penalties.py:89-92
      double g = p.p0;
      if (a <= mu) return 0.0;
      return a < g * mu ? g * (a - mu) / (g - 1.0) : a;
    }
    case 3: {  // penalties.py:135-139
      double s = p.p0;
      if (a <= 2.0 * mu) return fmax(a - mu, 0.0);
      return a <= s * mu ? ((s - 1.0) * a - s * mu) / (s - 2.0) : a;
    }
    case 4:
      return lq_prox_abs(p.p0, mu, a);
    case 5: {  // penalties.py:231-246: best of four candidates, ties -> smaller
      double q = p.p0, th = p.p1;
      double inner = lq_prox_abs(q, mu, a);
      double cand[4] = {0.0, inner < th ? inner : 0.0, th, a > th ? a : 0.0};
      double best = cand[0];
      double fb = pen_value(p, best, mu) + 0.5 * (best - a) * (best - a);
      for (int i = 1; i < 4; ++i) {
        double c = cand[i];
        double f = pen_value(p, c, mu) + 0.5 * (c - a) * (c - a);
        if (f < fb - 1e-15 || (fabs(f - fb) <= 1e-15 && c < best)) {
          best = c;
          fb = f;
        }
      }
      return best;
    }
    default: {  // penalties.py:262-270
      double g = p.p0;
      double disc = (a + g) * (a + g) - 4.0 * mu;
      double root = 0.0;
      if (disc >= 0) {
        root = 0.5 * ((a - g) + sqrt(fmax(disc, 0.0)));
        if (!(root > 0)) root = 0.0;
      }
      double fr = mu * log1p(root / g) + 0.5 * (root - a) * (root - a);
      return fr < 0.5 * a * a - 1e-15 ? root : 0.0;
    }
  }
}

// Signed prox (penalties.py:45-61): mu == 0 is the identity.
__host__ __device__ inline double prox(const Penalty& p, double mu, double v) {
  if (mu == 0.0) return v;
  double a = fabs(v);
  double r = prox_abs(p, mu, a);
  return v > 0 ? r : (v < 0 ? -r : 0.0);
}

}  // namespace tr
