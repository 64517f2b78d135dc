// Host cyclic Jacobi sweeps -- bit-exact restatement of the reference's
// numpy jacobi_eigh rotation loop (spectral.py:155-195).  Built with
// -ffp-contract=off so every product/sum rounds exactly like the numpy
// elementwise ufuncs; rounds use the circle-method schedule of
// spectral.py:114-131.  Pairs inside one round touch disjoint rows/columns,
// so they are applied in parallel (OpenMP) without changing any bit.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/taco_b200.h"

namespace taco {
void set_error(const char* fmt, ...);
}

namespace {

std::vector<std::vector<std::pair<int, int>>> circle_rounds(int d) {
  const int m = d + (d & 1);
  std::vector<int> ring(m);
  for (int i = 0; i < m; ++i) ring[i] = i;
  std::vector<std::vector<std::pair<int, int>>> out;
  for (int r = 0; r < m - 1; ++r) {
    std::vector<std::pair<int, int>> pr;
    for (int i = 0; i < m / 2; ++i) {
      int a = ring[i], b = ring[m - 1 - i];
      if (a < d && b < d) pr.emplace_back(a < b ? a : b, a < b ? b : a);
    }
    out.push_back(pr);
    std::vector<int> nx(m);
    nx[0] = ring[0];
    nx[1] = ring[m - 1];
    for (int i = 1; i < m - 1; ++i) nx[i + 1] = ring[i];
    ring.swap(nx);
  }
  return out;
}

double max_offdiag(const double* A, int d) {
  double mx = 0.0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      if (i != j) {
        double v = std::fabs(A[(size_t)i * d + j]);
        if (v > mx) mx = v;
      }
  return mx;
}

}  // namespace

extern "C" int taco_jacobi_sweeps(double* A, double* V, int32_t d, double tol, int32_t max_sweeps,
                                  int32_t* sweeps_out, double* residual_out) {
  if (d < 0) {
    taco::set_error("negative dimension");
    return TACO_ERR_PARAMETER;
  }
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) V[(size_t)i * d + j] = i == j ? 1.0 : 0.0;
  *sweeps_out = 0;
  *residual_out = 0.0;
  if (d <= 1) return TACO_OK;
  const auto rounds = circle_rounds(d);
  std::vector<int> P, Q;
  std::vector<double> C, S;
  bool converged = false;
  int sweeps = 0;
  for (int sw = 0; sw < max_sweeps; ++sw) {
    if (max_offdiag(A, d) <= tol) {
      converged = true;
      break;
    }
    ++sweeps;
    for (const auto& pr : rounds) {
      P.clear(); Q.clear(); C.clear(); S.clear();
      for (const auto& pq : pr) {
        const int p = pq.first, q = pq.second;
        const double apq = A[(size_t)p * d + q];
        if (apq == 0.0) continue;
        const double tau = (A[(size_t)q * d + q] - A[(size_t)p * d + p]) / (2.0 * apq);
        const double sg = tau < 0.0 ? -1.0 : 1.0;
        const double t = sg / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = t * c;
        P.push_back(p); Q.push_back(q); C.push_back(c); S.push_back(s);
      }
      const int np = (int)P.size();
      if (np == 0) continue;
      // rows: A[p,:] = c*Ap - s*Aq ; A[q,:] = s*Ap + c*Aq
#pragma omp parallel for schedule(static) if (np * d > 16384)
      for (int e = 0; e < np; ++e) {
        double* rp = A + (size_t)P[e] * d;
        double* rq = A + (size_t)Q[e] * d;
        const double c = C[e], s = S[e];
        for (int x = 0; x < d; ++x) {
          const double a = rp[x], b = rq[x];
          const double cp = c * a, sq = s * b, sp = s * a, cq = c * b;
          rp[x] = cp - sq;
          rq[x] = sp + cq;
        }
      }
      // columns: A[:,p] = Ap*c - Aq*s ; A[:,q] = Ap*s + Aq*c ; then V likewise
#pragma omp parallel for schedule(static) if (np * d > 16384)
      for (int r = 0; r < d; ++r) {
        double* ar = A + (size_t)r * d;
        double* vr = V + (size_t)r * d;
        for (int e = 0; e < np; ++e) {
          const int p = P[e], q = Q[e];
          const double c = C[e], s = S[e];
          const double a = ar[p], b = ar[q];
          const double ac = a * c, bs = b * s, as = a * s, bc = b * c;
          ar[p] = ac - bs;
          ar[q] = as + bc;
          const double va = vr[p], vb = vr[q];
          const double vac = va * c, vbs = vb * s, vas = va * s, vbc = vb * c;
          vr[p] = vac - vbs;
          vr[q] = vas + vbc;
        }
      }
      for (int e = 0; e < np; ++e) {
        A[(size_t)P[e] * d + Q[e]] = 0.0;
        A[(size_t)Q[e] * d + P[e]] = 0.0;
      }
    }
  }
  *sweeps_out = sweeps;
  if (!converged) {
    const double res = max_offdiag(A, d);
    *residual_out = res;
    if (res > tol) {
      taco::set_error("eigensolver hit the %d-sweep cap with off-diagonal residual %.3e above tolerance %.3e",
                      max_sweeps, res, tol);
      return TACO_ERR_CONVERGENCE;
    }
  }
  return TACO_OK;
}
