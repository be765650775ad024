// Host-side 1D constant tables for the kernels (basis setup, row a1):
// GLL nodes ("the p+1 Gauss-Lobatto points"), Gauss q = p+1 rule
// (reading c1), Lagrange values/derivatives, and the element-structured
// coarsening chain (reading c3).  Computed once per mesh in long
// double; p+1 numbers each, uploaded as kernel parameters.
#include <cmath>
#include <string>
#include <vector>

#include "common.h"

namespace lorpc {

static thread_local std::string g_err;
void set_error(const std::string& s) { g_err = s; }
int fail(int code, const std::string& s) { g_err = s; return code; }
const char* last_error() { return g_err.c_str(); }
long long& launch_counter() { static thread_local long long c = 0; return c; }

// (P_n(x), P_n'(x)) by the Bonnet recurrence, long double
static void leg(int n, long double x, long double& P, long double& dP) {
  long double a = 1.0L, b = x;
  if (n == 0) { P = 1.0L; dP = 0.0L; return; }
  for (int k = 2; k <= n; ++k) { long double c = ((2 * k - 1) * x * b - (k - 1) * a) / k; a = b; b = c; }
  P = b;
  dP = (std::fabs((double)x) < 1.0) ? n * (a - x * b) / (1.0L - x * x) : 0.5L * n * (n + 1) * (x > 0 ? 1.0L : ((n % 2) ? 1.0L : -1.0L));
}

void make_basis(int p, Basis1D& B, int quad) {
  B.p = p; B.q = p + 1;
  // GLL on [-1,1]: +-1 and the zeros of P_p'; Newton on P_p' with
  // (P_p')' = (2x P_p' - p(p+1) P_p) / (1 - x^2)
  long double t[MAXP + 1];
  t[0] = -1.0L; t[p] = 1.0L;
  for (int i = 1; i < p; ++i) {
    long double x = -std::cos(M_PI * (long double)i / p);
    for (int it = 0; it < 60; ++it) {
      long double P, dP; leg(p, x, P, dP);
      long double d2 = (2 * x * dP - (long double)p * (p + 1) * P) / (1.0L - x * x);
      long double dx = dP / d2; x -= dx;
      if (std::fabs((double)dx) < 1e-19) break;
    }
    t[i] = x;
  }
  for (int i = 0; i <= p; ++i) B.xi[i] = (double)(0.5L * (t[i] + 1.0L));
  for (int i = 0; i <= p / 2; ++i) { double a = 0.5 * (B.xi[i] + 1.0 - B.xi[p - i]); B.xi[i] = a; B.xi[p - i] = 1.0 - a; }
  B.xi[0] = 0.0; B.xi[p] = 1.0;
  // Gauss-Legendre q = p+1 on [0,1]
  const int q = p + 1;
  for (int i = 0; i < q; ++i) {
    long double x = -std::cos(M_PI * (i + 0.75L) / (q + 0.5L));
    for (int it = 0; it < 60; ++it) {
      long double P, dP; leg(q, x, P, dP);
      long double dx = P / dP; x -= dx;
      if (std::fabs((double)dx) < 1e-19) break;
    }
    long double P, dP; leg(q, x, P, dP);
    B.xq[i] = (double)(0.5L * (x + 1.0L));
    B.wq[i] = (double)(1.0L / ((1.0L - x * x) * dP * dP));
  }
  // Lagrange basis on the GLL nodes: barycentric weights, long double
  long double xl[MAXP + 1], bw[MAXP + 1];
  for (int j = 0; j <= p; ++j) xl[j] = B.xi[j];
  for (int j = 0; j <= p; ++j) {
    long double s = 1.0L;
    for (int k = 0; k <= p; ++k) if (k != j) s *= (xl[j] - xl[k]);
    bw[j] = 1.0L / s;
  }
  auto eval = [&](long double x, long double* val, long double* der) {
    // l_j(x) = prod_{k != j}(x - x_k) * bw_j ; l_j'(x) = l_j(x) * sum_{k != j} 1/(x - x_k),
    // evaluated without division by zero via explicit products
    for (int j = 0; j <= p; ++j) {
      long double v = bw[j], d = 0.0L;
      for (int k = 0; k <= p; ++k) if (k != j) v *= (x - xl[k]);
      for (int k = 0; k <= p; ++k) {
        if (k == j) continue;
        long double w = bw[j];
        for (int m = 0; m <= p; ++m) if (m != j && m != k) w *= (x - xl[m]);
        d += w;
      }
      val[j] = v; der[j] = d;
    }
  };
  if (quad == 1) {
    // GLL collocation: the rule's points are the nodes, w_i = 2 / (p (p+1) P_p(t_i)^2)
    // on [-1,1], halved on [0,1]
    for (int i = 0; i <= p; ++i) {
      long double P, dP;
      leg(p, t[i], P, dP);
      B.xq[i] = B.xi[i];
      B.wq[i] = (double)(1.0L / ((long double)p * (p + 1) * P * P));
    }
  }
  long double v[MAXP + 1], d[MAXP + 1];
  for (int i = 0; i < q; ++i) {
    eval(B.xq[i], v, d);
    for (int j = 0; j <= p; ++j) { B.B[i * (p + 1) + j] = (double)v[j]; B.D[i * (p + 1) + j] = (double)d[j]; }
    if (quad == 1)  // l_j(x_i) = delta_ij exactly
      for (int j = 0; j <= p; ++j) B.B[i * (p + 1) + j] = i == j ? 1.0 : 0.0;
  }
  eval(0.0L, v, d); for (int j = 0; j <= p; ++j) B.E0[j] = (double)d[j];
  eval(1.0L, v, d); for (int j = 0; j <= p; ++j) B.E1[j] = (double)d[j];
  // inverse of the reference 1D mass matrix M1 = B^T diag(w) B (Gauss-Jordan, long double)
  const int m = p + 1;
  long double A[MAXP + 1][2 * (MAXP + 1)];
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      long double s = 0.0L;
      for (int k = 0; k < q; ++k) s += (long double)B.wq[k] * B.B[k * m + i] * B.B[k * m + j];
      A[i][j] = s;
      A[i][m + j] = (i == j) ? 1.0L : 0.0L;
    }
  for (int c = 0; c < m; ++c) {
    int piv = c;
    for (int r = c + 1; r < m; ++r) if (std::fabs((double)A[r][c]) > std::fabs((double)A[piv][c])) piv = r;
    for (int j = 0; j < 2 * m; ++j) std::swap(A[c][j], A[piv][j]);
    const long double inv = 1.0L / A[c][c];
    for (int j = 0; j < 2 * m; ++j) A[c][j] *= inv;
    for (int r = 0; r < m; ++r) {
      if (r == c) continue;
      const long double f = A[r][c];
      for (int j = 0; j < 2 * m; ++j) A[r][j] -= f * A[c][j];
    }
  }
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) B.M1inv[i * m + j] = (double)A[i][m + j];
}

std::vector<std::vector<int>> make_chain(int p) {
  // keep both end points, drop every other interior point left to right
  // (odd 1-based interior positions), until no interior point remains
  std::vector<std::vector<int>> out(1);
  for (int i = 0; i <= p; ++i) out[0].push_back(i);
  while (out.back().size() > 2) {
    const std::vector<int>& c = out.back();
    std::vector<int> nx{c.front()};
    for (size_t t = 2; t + 1 < c.size(); t += 2) nx.push_back(c[t]);
    nx.push_back(c.back());
    out.push_back(nx);
  }
  return out;
}

}  // namespace lorpc
