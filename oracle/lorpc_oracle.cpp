// =============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, deliberately unoptimised CPU implementation of what the
// paper's PCG hot path computes (arXiv 1908.07071, "Matrix-free preconditioners
// for high-order continuous and discontinuous Galerkin discretizations").
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load this library.  It shares no code, header, table or
// constant generator with the CUDA product (paper_1908_07071_b200/csrc).
//
// Citations: "P:n" = /root/reference/PAPER.md line n (section / \label named),
// "S:n" = SPEC.md line n; readings "cN" = DESIGN.md §Readings.
//
// What it does, in the paper's order:
//   basis  -> mesh / element maps
//   -> explicitly assembled element stiffness K_e and y = sum_e P_e^T K_e P_e x
//      (eq:fem P:86-89, eq:system P:95-97)
//   -> LOR stiffness K_h on the GLL-refined mesh
//   -> element-structured hierarchy, Galerkin levels (reading c3/c4)
//   -> vertex / element-star patches (eq:patch P:302-315, reading c9)
//   -> MDF-ordered ILU(0) per patch and level (readings c5/c6)
//   -> V(1,1) cycle per patch, dense Cholesky at the coarsest level
//   -> coarse space V_0 = Q1 on T_p, R_0 = GMG V(1,1) with l1-Jacobi (P:289-300,
//      reading c11)
//   -> additive Schwarz B = sum_j R_j Q_j (eq:as P:274-277)
//   -> PCG (reading c12)
//   -> SIPG DG operator (eq:ip P:113-136) and B_DG (eq:dg-as P:635-641)
//
// Floating point: FP64 everywhere, built with -O2 -ffp-contract=off.  OpenMP
// is used only across independent elements / patches; every reduction that
// combines their results is done afterwards in a fixed (ascending) order.
//
// Parity status per function: see DESIGN.md "Oracle pins".  The MDF ordering
// on perturbed meshes is "parity unpinned beyond the validity rule" (c6).
// =============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef std::vector<double> vec;
typedef int64_t i64;

static std::string g_err;
extern "C" const char* or_last_error() { return g_err.c_str(); }

// -----------------------------------------------------------------------------
// 1. One-dimensional basis on the reference interval [0,1]
// -----------------------------------------------------------------------------
// Legendre polynomial P_n and its derivative by the three-term recurrence.
static void legendre(int n, double x, double* P, double* dP) {
  double p0 = 1.0, p1 = x;
  if (n == 0) { *P = 1.0; *dP = 0.0; return; }
  for (int k = 2; k <= n; ++k) {
    double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1; p1 = p2;
  }
  *P = p1;
  // P_n'(x) = n (x P_n - P_{n-1}) / (x^2 - 1), valid for |x| < 1
  *dP = n * (x * p1 - p0) / (x * x - 1.0);
}

// Gauss-Lobatto-Legendre nodes/weights: endpoints plus the roots of P_p'
// (Newton on P_p' from Chebyshev-Lobatto guesses), mapped to [0,1].
static void gll_rule(int p, vec& x, vec& w) {
  x.assign(p + 1, 0.0); w.assign(p + 1, 0.0);
  std::vector<double> t(p + 1);
  t[0] = -1.0; t[p] = 1.0;
  for (int i = 1; i < p; ++i) {
    double z = -std::cos(M_PI * i / p);
    for (int it = 0; it < 100; ++it) {
      double P, dP; legendre(p, z, &P, &dP);
      // Legendre ODE: (1 - z^2) P'' = 2 z P' - p(p+1) P
      double d2P = (2.0 * z * dP - p * (p + 1.0) * P) / (1.0 - z * z);
      double dz = dP / d2P;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    t[i] = z;
  }
  for (int i = 0; i <= p; ++i) {
    double P, dP;
    if (i == 0 || i == p) P = (i == 0) ? ((p % 2) ? -1.0 : 1.0) : 1.0;
    else legendre(p, t[i], &P, &dP);
    w[i] = 2.0 / (p * (p + 1.0) * P * P) / 2.0;  // /2: length of [0,1]
  }
  for (int i = 0; i <= p; ++i) x[i] = 0.5 * (t[i] + 1.0);
  // exact symmetry about 1/2: average mirrored pairs
  for (int i = 0; i <= p / 2; ++i) {
    double a = 0.5 * (x[i] + (1.0 - x[p - i]));
    x[i] = a; x[p - i] = 1.0 - a;
    double b = 0.5 * (w[i] + w[p - i]);
    w[i] = b; w[p - i] = b;
  }
  x[0] = 0.0; x[p] = 1.0;
}

// Gauss-Legendre q-point rule on [0,1] (Newton on P_q).  Reading c1.
static void gauss_rule(int q, vec& x, vec& w) {
  x.assign(q, 0.0); w.assign(q, 0.0);
  for (int i = 0; i < q; ++i) {
    double z = -std::cos(M_PI * (i + 0.75) / (q + 0.5));
    for (int it = 0; it < 100; ++it) {
      double P, dP; legendre(q, z, &P, &dP);
      double dz = P / dP;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    double P, dP; legendre(q, z, &P, &dP);
    x[i] = 0.5 * (z + 1.0);
    w[i] = 2.0 / ((1.0 - z * z) * dP * dP) / 2.0;
  }
  for (int i = 0; i < q / 2; ++i) {
    double a = 0.5 * (x[i] + (1.0 - x[q - 1 - i]));
    x[i] = a; x[q - 1 - i] = 1.0 - a;
    double b = 0.5 * (w[i] + w[q - 1 - i]);
    w[i] = b; w[q - 1 - i] = b;
  }
  if (q % 2) x[q / 2] = 0.5;
}

// Nodal Lagrange basis l_j on nodes xn, and its derivative, at a point t.
static double lagrange(const vec& xn, int j, double t) {
  double v = 1.0;
  for (size_t m = 0; m < xn.size(); ++m)
    if ((int)m != j) v *= (t - xn[m]) / (xn[j] - xn[m]);
  return v;
}
static double dlagrange(const vec& xn, int j, double t) {
  double s = 0.0;
  for (size_t k = 0; k < xn.size(); ++k) {
    if ((int)k == j) continue;
    double v = 1.0 / (xn[j] - xn[k]);
    for (size_t m = 0; m < xn.size(); ++m)
      if ((int)m != j && m != k) v *= (t - xn[m]) / (xn[j] - xn[m]);
    s += v;
  }
  return s;
}

struct Basis {
  int p, q;
  vec xi, wgll;  // GLL nodes / weights on [0,1]
  vec xg, wg;    // volume rule on [0,1], q = p+1 points: Gauss (reading c1) or, with
                 // quad = 1, the GLL nodes themselves (collocation)
  vec B, D;      // [q][p+1]: l_j(xg_i), l_j'(xg_i)
  void init(int p_, int quad = 0) {
    p = p_; q = p + 1;
    gll_rule(p, xi, wgll);
    if (quad == 1) { xg = xi; wg = wgll; }
    else gauss_rule(q, xg, wg);
    B.assign(q * (p + 1), 0.0); D.assign(q * (p + 1), 0.0);
    for (int i = 0; i < q; ++i)
      for (int j = 0; j <= p; ++j) {
        B[i * (p + 1) + j] = lagrange(xi, j, xg[i]);
        D[i * (p + 1) + j] = dlagrange(xi, j, xg[i]);
      }
  }
};

extern "C" int or_basis(int p, double* xi, double* wgll, double* xg, double* wg,
                        double* B, double* D) {
  if (p < 1) { g_err = "basis: p must be >= 1"; return 1; }
  Basis b; b.init(p);
  std::copy(b.xi.begin(), b.xi.end(), xi);
  std::copy(b.wgll.begin(), b.wgll.end(), wgll);
  std::copy(b.xg.begin(), b.xg.end(), xg);
  std::copy(b.wg.begin(), b.wg.end(), wg);
  std::copy(b.B.begin(), b.B.end(), B);
  std::copy(b.D.begin(), b.D.end(), D);
  return 0;
}

// -----------------------------------------------------------------------------
// 2. Small dense linear algebra helpers
// -----------------------------------------------------------------------------
static double det_inv(int d, const double* J, double* Ji) {
  if (d == 2) {
    double det = J[0] * J[3] - J[1] * J[2];
    Ji[0] = J[3] / det; Ji[1] = -J[1] / det; Ji[2] = -J[2] / det; Ji[3] = J[0] / det;
    return det;
  }
  double det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
               J[2] * (J[3] * J[7] - J[4] * J[6]);
  Ji[0] = (J[4] * J[8] - J[5] * J[7]) / det;
  Ji[1] = (J[2] * J[7] - J[1] * J[8]) / det;
  Ji[2] = (J[1] * J[5] - J[2] * J[4]) / det;
  Ji[3] = (J[5] * J[6] - J[3] * J[8]) / det;
  Ji[4] = (J[0] * J[8] - J[2] * J[6]) / det;
  Ji[5] = (J[2] * J[3] - J[0] * J[5]) / det;
  Ji[6] = (J[3] * J[7] - J[4] * J[6]) / det;
  Ji[7] = (J[1] * J[6] - J[0] * J[7]) / det;
  Ji[8] = (J[0] * J[4] - J[1] * J[3]) / det;
  return det;
}

// Dense Cholesky A = C C^T in place (lower), returns false if not SPD.
static bool cholesky(int n, vec& A) {
  for (int j = 0; j < n; ++j) {
    double s = A[j * n + j];
    for (int k = 0; k < j; ++k) s -= A[j * n + k] * A[j * n + k];
    if (!(s > 0.0)) return false;
    double c = std::sqrt(s);
    A[j * n + j] = c;
    for (int i = j + 1; i < n; ++i) {
      double t = A[i * n + j];
      for (int k = 0; k < j; ++k) t -= A[i * n + k] * A[j * n + k];
      A[i * n + j] = t / c;
    }
  }
  return true;
}
static void chol_solve(int n, const vec& C, double* x) {
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int k = 0; k < i; ++k) s -= C[i * n + k] * x[k];
    x[i] = s / C[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int k = i + 1; k < n; ++k) s -= C[k * n + i] * x[k];
    x[i] = s / C[i * n + i];
  }
}

// -----------------------------------------------------------------------------
// 3. Compressed sparse row matrices (plain; sorted column indices)
// -----------------------------------------------------------------------------
struct CSR {
  i64 nr = 0, nc = 0;
  std::vector<i64> rp;
  std::vector<int> ci;
  vec v;
  i64 nnz() const { return (i64)ci.size(); }
  double get(i64 i, int j) const {
    auto b = ci.begin() + rp[i], e = ci.begin() + rp[i + 1];
    auto it = std::lower_bound(b, e, j);
    if (it != e && *it == j) return v[it - ci.begin()];
    return 0.0;
  }
  void matvec(const double* x, double* y) const {
    for (i64 i = 0; i < nr; ++i) {
      double s = 0.0;
      for (i64 k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
      y[i] = s;
    }
  }
};

struct Trip { i64 r; int c; double v; };

// Triplets -> CSR, duplicates summed in the order they appear after a stable sort.
static CSR csr_from_triplets(i64 nr, i64 nc, std::vector<Trip>& t) {
  std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
    return a.r < b.r || (a.r == b.r && a.c < b.c);
  });
  CSR A; A.nr = nr; A.nc = nc; A.rp.assign(nr + 1, 0);
  for (size_t k = 0; k < t.size();) {
    size_t e = k; double s = 0.0;
    while (e < t.size() && t[e].r == t[k].r && t[e].c == t[k].c) { s += t[e].v; ++e; }
    A.ci.push_back(t[k].c); A.v.push_back(s); A.rp[t[k].r + 1]++;
    k = e;
  }
  for (i64 i = 0; i < nr; ++i) A.rp[i + 1] += A.rp[i];
  return A;
}

static CSR csr_transpose(const CSR& A) {
  CSR T; T.nr = A.nc; T.nc = A.nr; T.rp.assign(T.nr + 1, 0);
  for (i64 k = 0; k < A.nnz(); ++k) T.rp[A.ci[k] + 1]++;
  for (i64 i = 0; i < T.nr; ++i) T.rp[i + 1] += T.rp[i];
  T.ci.resize(A.nnz()); T.v.resize(A.nnz());
  std::vector<i64> pos(T.rp.begin(), T.rp.end() - 1);
  for (i64 i = 0; i < A.nr; ++i)
    for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
      i64 d = pos[A.ci[k]]++;
      T.ci[d] = (int)i; T.v[d] = A.v[k];
    }
  return T;
}

// C = A * B (row-by-row sparse accumulator).
static CSR csr_mult(const CSR& A, const CSR& B) {
  CSR C; C.nr = A.nr; C.nc = B.nc; C.rp.assign(A.nr + 1, 0);
  std::vector<double> acc(B.nc, 0.0);
  std::vector<char> used(B.nc, 0);
  std::vector<int> cols;
  for (i64 i = 0; i < A.nr; ++i) {
    cols.clear();
    for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
      int a = A.ci[k]; double av = A.v[k];
      for (i64 l = B.rp[a]; l < B.rp[a + 1]; ++l) {
        int c = B.ci[l];
        if (!used[c]) { used[c] = 1; cols.push_back(c); acc[c] = 0.0; }
        acc[c] += av * B.v[l];
      }
    }
    std::sort(cols.begin(), cols.end());
    for (int c : cols) { C.ci.push_back(c); C.v.push_back(acc[c]); used[c] = 0; }
    C.rp[i + 1] = (i64)C.ci.size();
  }
  return C;
}

// Galerkin product P^T A P (reading c4).
static CSR galerkin(const CSR& A, const CSR& P) {
  CSR AP = csr_mult(A, P);
  CSR Pt = csr_transpose(P);
  return csr_mult(Pt, AP);
}

// Restriction of A to index subsets (rows `ri`, cols `cj`; global->local maps).
static CSR csr_submatrix(const CSR& A, const std::vector<i64>& ri, const std::vector<i64>& cj) {
  std::map<i64, int> cmap;
  for (size_t k = 0; k < cj.size(); ++k) cmap[cj[k]] = (int)k;
  std::vector<Trip> t;
  for (size_t r = 0; r < ri.size(); ++r)
    for (i64 k = A.rp[ri[r]]; k < A.rp[ri[r] + 1]; ++k) {
      auto it = cmap.find(A.ci[k]);
      if (it != cmap.end()) t.push_back({(i64)r, it->second, A.v[k]});
    }
  return csr_from_triplets((i64)ri.size(), (i64)cj.size(), t);
}

// -----------------------------------------------------------------------------
// 4. Mesh of tensor-product elements; each element is the image of [0,1]^d under
//    the multilinear map of its 2^d vertices.  Cartesian topology
//    n0 x n1 (x n2), vertices x-fastest; CG dofs = global GLL node grid
//    (np+1)^d, Dirichlet = grid boundary.
// -----------------------------------------------------------------------------
struct Problem;

struct Mesh {
  int d = 2, p = 1;
  int n[3] = {1, 1, 1};   // elements per axis (n[2] = 1 in 2D)
  int N[3] = {1, 1, 1};   // GLL nodes per axis: n p + 1 (1 in unused axis)
  int nvx[3] = {1, 1, 1}; // vertices per axis
  i64 nel = 0, ndof = 0, nvert = 0;
  vec V;                  // [nvert][d]
  Basis b;
  // variable coefficient b(x) of -div(b grad u) (sec:variable-coeff; row
  // f3), sampled by the harness: bq[e][iq] at the volume Gauss points (or_quad_points
  // layout), bs[sub][ig] at the 2^d Gauss points of every LOR subcell (global subcell
  // index sx + (N0-1)(sy + (N1-1) sz), or_subcell_points layout).  Empty: b = 1.
  vec bq, bs;
  i64 sub_index(const int* sg) const { return sg[0] + (i64)(N[0] - 1) * (sg[1] + (i64)(N[1] - 1) * sg[2]); }

  void elem_coords(i64 e, int* ec) const {
    ec[0] = (int)(e % n[0]); i64 r = e / n[0];
    ec[1] = (int)(r % n[1]); ec[2] = (int)(r / n[1]);
    if (d == 2) ec[2] = 0;
  }
  i64 node_index(const int* g) const { return g[0] + (i64)N[0] * (g[1] + (i64)N[1] * g[2]); }
  bool is_dirichlet(i64 g) const {
    int c[3] = {(int)(g % N[0]), (int)((g / N[0]) % N[1]), (int)(g / ((i64)N[0] * N[1]))};
    for (int k = 0; k < d; ++k)
      if (c[k] == 0 || c[k] == N[k] - 1) return true;
    return false;
  }
  int nloc() const { return d == 2 ? (p + 1) * (p + 1) : (p + 1) * (p + 1) * (p + 1); }
  // local node a -> (a0,a1,a2), x-fastest
  void local_coords(int a, int* lc) const {
    lc[0] = a % (p + 1); lc[1] = (a / (p + 1)) % (p + 1); lc[2] = (d == 3) ? a / ((p + 1) * (p + 1)) : 0;
  }
  i64 l2g(i64 e, int a) const {
    int ec[3], lc[3], g[3] = {0, 0, 0};
    elem_coords(e, ec); local_coords(a, lc);
    for (int k = 0; k < d; ++k) g[k] = ec[k] * p + lc[k];
    return node_index(g);
  }
  // multilinear element map x(xi) and its Jacobian J[i][k] = dx_i / dxi_k
  void map(i64 e, const double* xi, double* x, double* J) const {
    int ec[3]; elem_coords(e, ec);
    for (int i = 0; i < d; ++i) { x[i] = 0.0; for (int k = 0; k < d; ++k) J[i * d + k] = 0.0; }
    int nc = 1 << d;
    for (int c = 0; c < nc; ++c) {
      int cb[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
      int vg[3] = {ec[0] + cb[0], ec[1] + cb[1], d == 3 ? ec[2] + cb[2] : 0};
      i64 vid = vg[0] + (i64)nvx[0] * (vg[1] + (i64)nvx[1] * vg[2]);
      double phi[3], dphi[3];
      for (int k = 0; k < d; ++k) {
        phi[k] = cb[k] ? xi[k] : 1.0 - xi[k];
        dphi[k] = cb[k] ? 1.0 : -1.0;
      }
      double s = 1.0;
      for (int k = 0; k < d; ++k) s *= phi[k];
      for (int i = 0; i < d; ++i) x[i] += V[vid * d + i] * s;
      for (int k = 0; k < d; ++k) {
        double g = dphi[k];
        for (int m = 0; m < d; ++m) if (m != k) g *= phi[m];
        for (int i = 0; i < d; ++i) J[i * d + k] += V[vid * d + i] * g;
      }
    }
  }
};

// Element stiffness, explicitly assembled (eq:fem P:86-89):
//   K_e[a][b] = sum_q wq detJ_q (J_q^{-T} grad phi_a)(q) . (J_q^{-T} grad phi_b)(q)
// with Gauss q=p+1 per direction (reading c1).  Returns false on det J <= 0.
static bool elem_stiffness(const Mesh& m, i64 e, vec& K) {
  const int d = m.d, p = m.p, q = m.b.q, nl = m.nloc();
  int nq = (d == 2) ? q * q : q * q * q;
  K.assign((size_t)nl * nl, 0.0);
  std::vector<double> gr((size_t)nl * d), Gg((size_t)nl * d);
  for (int iq = 0; iq < nq; ++iq) {
    int qc[3] = {iq % q, (iq / q) % q, d == 3 ? iq / (q * q) : 0};
    double xi[3], x[3], J[9], Ji[9];
    double w = 1.0;
    for (int k = 0; k < d; ++k) { xi[k] = m.b.xg[qc[k]]; w *= m.b.wg[qc[k]]; }
    m.map(e, xi, x, J);
    double det = det_inv(d, J, Ji);
    if (!(det > 0.0)) { g_err = "inverted element " + std::to_string(e); return false; }
    // reference gradients of every nodal basis function at this point
    for (int a = 0; a < nl; ++a) {
      int lc[3]; m.local_coords(a, lc);
      for (int k = 0; k < d; ++k) {
        double g = 1.0;
        for (int mm = 0; mm < d; ++mm) {
          int idx = qc[mm] * (p + 1) + lc[mm];
          g *= (mm == k) ? m.b.D[idx] : m.b.B[idx];
        }
        gr[a * d + k] = g;
      }
      // physical gradient: J^{-T} grad_ref
      for (int i = 0; i < d; ++i) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) s += Ji[k * d + i] * gr[a * d + k];
        Gg[a * d + i] = s;
      }
    }
    double f = w * det;
    if (!m.bq.empty()) f *= m.bq[(size_t)e * nq + iq];   // b(x_q) (sec:variable-coeff)
    for (int a = 0; a < nl; ++a)
      for (int bb = 0; bb < nl; ++bb) {
        double s = 0.0;
        for (int i = 0; i < d; ++i) s += Gg[a * d + i] * Gg[bb * d + i];
        K[(size_t)a * nl + bb] += f * s;
      }
  }
  return true;
}

// -----------------------------------------------------------------------------
// 5. Problem handle
// -----------------------------------------------------------------------------
struct PatchLevel {
  int n = 0;                      // free nodes of the patch at this level
  std::vector<i64> gid;           // their level-global indices
  CSR A;                          // A_l restricted (reading c4)
  CSR P;                          // prolongation from level l+1 (patch restricted)
  std::vector<int> order, pos;    // MDF order (reading c6), inverse
  vec Lv;                         // L values aligned with A's CSR slots (lower entries)
  vec Dg;                         // pivots D_k
  vec C;                          // dense Cholesky factor at the coarsest level (c8)
  bool coarsest = false;
};
struct Patch { int elo[3], ehi[3]; std::vector<PatchLevel> lv; };

struct Problem {
  Mesh m;
  int disc = 0;           // 0 = CG, 1 = SIPG
  double eta = 0.0;       // SIPG penalty coefficient: sigma_e = eta / h_e (reading c13)
  int patch_kind = 0;     // 0 = vertex (eq:patch), 1 = element star (reading c9)
  int ordering = 0;       // 0 = MDF, 1 = natural, 2 = RCM (reading r5)
  int coarse = 0;         // 0 = GMG l1-Jacobi R_0 (reading c11), 1 = none, 2 = exact (dense)
  int local_exact = 0;    // 1: R_j = A_j^{-1} (dense Cholesky) instead of the V-cycle (pins only)
  int extend = 0;         // 1: vertex patches extended for isotropic overlap (sec:aniso, reading r6)
  std::vector<vec> Kel;   // cached element matrices (CG) or empty
  bool cached = false;
  // LOR and hierarchy
  std::vector<std::vector<int>> chain;  // retained GLL local indices per level (c3)
  std::vector<int> Nl;                  // nodes per axis at each level (per unit: m_l)
  std::vector<CSR> Al;                  // global level operators, full node grid
  std::vector<CSR> Pl;                  // P_l : level l+1 -> level l
  bool lor_built = false;
  std::vector<Patch> patches;
  bool schwarz_built = false;
  // coarse space
  CSR P0;                               // vertex grid -> LOR nodes (multilinear in reference coords)
  std::vector<i64> cfree;               // interior vertex ids
  std::vector<CSR> Ac;                  // GMG level operators (interior nodes only)
  std::vector<CSR> Pc;                  // GMG prolongations (interior only)
  std::vector<vec> dl1;                 // l1-Jacobi diagonals
  std::vector<std::vector<int>> cn;     // vertices per axis at each GMG level
  vec Cc; int ncc = 0;                  // coarsest exact solve (dense Cholesky)
  vec C0dense; int n0dense = 0;         // coarse=2: exact A_0 solve
  // DG
  vec DB;                               // diag(A_IP) (full DG vector)
  std::vector<vec> br2C;                // BR2: Cholesky factors of the element mass matrices
};

extern "C" void* or_create(int d, int n0, int n1, int n2, int p, const double* vertices) {
  if (d != 2 && d != 3) { g_err = "dim must be 2 or 3"; return nullptr; }
  if (p < 1 || n0 < 1 || n1 < 1 || (d == 3 && n2 < 1)) { g_err = "bad sizes"; return nullptr; }
  Problem* P = new Problem();
  Mesh& m = P->m;
  m.d = d; m.p = p; m.n[0] = n0; m.n[1] = n1; m.n[2] = (d == 3) ? n2 : 1;
  for (int k = 0; k < 3; ++k) {
    m.N[k] = (k < d) ? m.n[k] * p + 1 : 1;
    m.nvx[k] = (k < d) ? m.n[k] + 1 : 1;
  }
  m.nel = (i64)m.n[0] * m.n[1] * m.n[2];
  m.ndof = (i64)m.N[0] * m.N[1] * m.N[2];
  m.nvert = (i64)m.nvx[0] * m.nvx[1] * m.nvx[2];
  m.V.assign(vertices, vertices + m.nvert * d);
  m.b.init(p);
  return P;
}
extern "C" void or_destroy(void* h) { delete (Problem*)h; }

// Volume quadrature: 0 = Gauss q = p+1 (reading c1), 1 = GLL collocation (the
// quadrature points are the nodes; row f2's quadrature variant).  CG only.
extern "C" int or_set_quad(void* h, int quad) {
  Problem* P = (Problem*)h;
  if (quad != 0 && quad != 1) { g_err = "quad must be 0 or 1"; return 1; }
  if (quad == 1 && P->disc != 0) { g_err = "GLL collocation: CG only"; return 1; }
  P->m.b.init(P->m.p, quad);
  P->Kel.clear(); P->cached = false;
  return 0;
}

extern "C" int or_set_dg(void* h, int disc, double eta) {
  Problem* P = (Problem*)h;
  if (disc != 0 && !(eta > 0.0)) { g_err = "dg: eta must be > 0"; return 1; }
  P->disc = disc; P->eta = eta; return 0;
}

extern "C" i64 or_ndof(void* h) { return ((Problem*)h)->m.ndof; }

// Variable coefficient (row f3): bq [nquad] at the volume Gauss points, bs [nsub][2^d]
// at the LOR subcell Gauss points (either may be NULL = 1).  CG only.  Invalidates the
// cached element matrices, the LOR hierarchy and the Schwarz setup.
extern "C" i64 or_nsub(void* h) {
  const Mesh& m = ((Problem*)h)->m;
  i64 n = 1;
  for (int k = 0; k < m.d; ++k) n *= m.N[k] - 1;
  return n;
}
extern "C" int or_set_coefficient(void* h, const double* bq, const double* bs) {
  Problem* P = (Problem*)h;
  Mesh& m = P->m;
  if (P->disc != 0) { g_err = "coefficient: CG only"; return 1; }
  const int q = m.b.q, nq = m.d == 2 ? q * q : q * q * q;
  if (bq) m.bq.assign(bq, bq + m.nel * nq); else m.bq.clear();
  if (bs) m.bs.assign(bs, bs + or_nsub(h) * (1 << m.d)); else m.bs.clear();
  for (double v : m.bq) if (!(v > 0.0)) { g_err = "coefficient: b <= 0"; return 1; }
  for (double v : m.bs) if (!(v > 0.0)) { g_err = "coefficient: b <= 0"; return 1; }
  P->Kel.clear(); P->cached = false;
  P->lor_built = false; P->schwarz_built = false;
  return 0;
}
// Gauss points of every LOR subcell: X[sub][ig][d], the subcell map multilinear in
// the images of its corner GLL nodes (reading c2), t = 1/2 -+ 1/(2 sqrt 3).
extern "C" void or_subcell_points(void* h, double* X) {
  const Mesh& m = ((Problem*)h)->m;
  const int d = m.d, p = m.p, nc = 1 << d;
  const double gp[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
  const int nsub = d == 2 ? p * p : p * p * p;
  for (i64 e = 0; e < m.nel; ++e)
    for (int s = 0; s < nsub; ++s) {
      int sc[3] = {s % p, (s / p) % p, (d == 3) ? s / (p * p) : 0}, ec[3], sg[3] = {0, 0, 0};
      m.elem_coords(e, ec);
      for (int k = 0; k < d; ++k) sg[k] = ec[k] * p + sc[k];
      double Xc[8][3];
      for (int c = 0; c < nc; ++c) {
        double xi[3], x[3], J[9];
        for (int k = 0; k < d; ++k) xi[k] = m.b.xi[sc[k] + ((c >> k) & 1)];
        m.map(e, xi, x, J);
        for (int k = 0; k < d; ++k) Xc[c][k] = x[k];
      }
      for (int ig = 0; ig < nc; ++ig) {
        double* o = X + ((size_t)m.sub_index(sg) * nc + ig) * d;
        for (int i = 0; i < d; ++i) o[i] = 0.0;
        for (int c = 0; c < nc; ++c) {
          double wv = 1.0;
          for (int k = 0; k < d; ++k) {
            const double t = gp[(ig >> k) & 1];
            wv *= ((c >> k) & 1) ? t : 1.0 - t;
          }
          for (int i = 0; i < d; ++i) o[i] += wv * Xc[c][i];
        }
      }
    }
}

// Element stiffness matrix for tests.
extern "C" int or_elem_matrix(void* h, i64 e, double* out) {
  Problem* P = (Problem*)h; vec K;
  if (!elem_stiffness(P->m, e, K)) return 1;
  std::copy(K.begin(), K.end(), out);
  return 0;
}

static bool build_elem_cache(Problem* P) {
  if (P->cached) return true;
  const Mesh& m = P->m;
  P->Kel.assign(m.nel, vec());
  bool ok = true;
#pragma omp parallel for schedule(dynamic, 16)
  for (i64 e = 0; e < m.nel; ++e)
    if (!elem_stiffness(m, e, P->Kel[e])) ok = false;
  P->cached = ok;
  return ok;
}

// Physical coordinates of the CG nodes (images of the GLL grid).
extern "C" void or_node_coords(void* h, double* X) {
  const Mesh& m = ((Problem*)h)->m;
  for (i64 e = 0; e < m.nel; ++e)
    for (int a = 0; a < m.nloc(); ++a) {
      int lc[3]; m.local_coords(a, lc);
      double xi[3] = {m.b.xi[lc[0]], m.b.xi[lc[1]], m.b.xi[lc[2]]}, x[3], J[9];
      m.map(e, xi, x, J);
      i64 g = m.l2g(e, a);
      for (int k = 0; k < m.d; ++k) X[g * m.d + k] = x[k];
    }
}

// -----------------------------------------------------------------------------
// 6. CG operator  y = K_p x  with symmetric Dirichlet elimination:
//    y_F = K_FF x_F, y_D = x_D.  Element matrices are assembled explicitly
//    (north_star: "assembles the high-order matrix explicitly").
// -----------------------------------------------------------------------------
static void cg_apply(Problem* P, const double* x, double* y) {
  const Mesh& m = P->m;
  const int nl = m.nloc();
  std::vector<double> xm(x, x + m.ndof);
  for (i64 g = 0; g < m.ndof; ++g) if (m.is_dirichlet(g)) xm[g] = 0.0;
  std::fill(y, y + m.ndof, 0.0);
  vec Kt;
  for (i64 e = 0; e < m.nel; ++e) {
    const vec* K;
    if (P->cached) K = &P->Kel[e];
    else { elem_stiffness(m, e, Kt); K = &Kt; }
    for (int a = 0; a < nl; ++a) {
      double s = 0.0;
      for (int bb = 0; bb < nl; ++bb) s += (*K)[(size_t)a * nl + bb] * xm[m.l2g(e, bb)];
      y[m.l2g(e, a)] += s;
    }
  }
  for (i64 g = 0; g < m.ndof; ++g) if (m.is_dirichlet(g)) y[g] = x[g];
}

// Rows of y = K_p x for sampled nodes only (full-size parity on samples).
extern "C" int or_apply_K_rows(void* h, const double* x, const i64* rows, i64 nrows, double* out) {
  Problem* P = (Problem*)h; const Mesh& m = P->m;
  const int d = m.d, p = m.p, nl = m.nloc();
  for (i64 r = 0; r < nrows; ++r) {
    i64 g = rows[r];
    if (m.is_dirichlet(g)) { out[r] = x[g]; continue; }
    int gc[3] = {(int)(g % m.N[0]), (int)((g / m.N[0]) % m.N[1]), (int)(g / ((i64)m.N[0] * m.N[1]))};
    double s = 0.0;
    // every element containing node g, in ascending element order
    int lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
      if (k >= d) { lo[k] = hi[k] = 0; continue; }
      lo[k] = std::max(0, (gc[k] - 1) / p); hi[k] = std::min(m.n[k] - 1, gc[k] / p);
      if (gc[k] == 0) lo[k] = 0;
    }
    for (int ez = lo[2]; ez <= hi[2]; ++ez)
      for (int ey = lo[1]; ey <= hi[1]; ++ey)
        for (int ex = lo[0]; ex <= hi[0]; ++ex) {
          int ec[3] = {ex, ey, ez};
          bool in = true; int a = 0, mul = 1;
          for (int k = 0; k < d; ++k) {
            int lcv = gc[k] - ec[k] * p;
            if (lcv < 0 || lcv > p) in = false;
            a += lcv * mul; mul *= (p + 1);
          }
          if (!in) continue;
          i64 e = ex + (i64)m.n[0] * (ey + (i64)m.n[1] * ez);
          vec K;
          if (P->cached) K = P->Kel[e]; else elem_stiffness(m, e, K);
          for (int bb = 0; bb < nl; ++bb) {
            i64 gb = m.l2g(e, bb);
            if (!m.is_dirichlet(gb)) s += K[(size_t)a * nl + bb] * x[gb];
          }
        }
    out[r] = s;
  }
  return 0;
}

// -----------------------------------------------------------------------------
// 7. Right-hand side (f, v) by Gauss quadrature (eq:fem); Dirichlet rows zeroed.
//    The harness evaluates f at the points returned by or_quad_points.
// -----------------------------------------------------------------------------
extern "C" i64 or_nquad(void* h) {
  const Mesh& m = ((Problem*)h)->m;
  return m.nel * (m.d == 2 ? m.b.q * m.b.q : m.b.q * m.b.q * m.b.q);
}
extern "C" void or_quad_points(void* h, double* X) {
  const Mesh& m = ((Problem*)h)->m; const int d = m.d, q = m.b.q;
  int nq = (d == 2) ? q * q : q * q * q;
  for (i64 e = 0; e < m.nel; ++e)
    for (int iq = 0; iq < nq; ++iq) {
      int qc[3] = {iq % q, (iq / q) % q, iq / (q * q)};
      double xi[3], x[3], J[9];
      for (int k = 0; k < d; ++k) xi[k] = m.b.xg[qc[k]];
      m.map(e, xi, x, J);
      for (int k = 0; k < d; ++k) X[(e * nq + iq) * d + k] = x[k];
    }
}
// b_i = sum_e sum_q w_q detJ_q f(x_q) phi_i(x_q); `dg` selects element-major DG layout.
extern "C" int or_rhs(void* h, const double* fq, double* b, int dg) {
  Problem* P = (Problem*)h; const Mesh& m = P->m; const int d = m.d, p = m.p, q = m.b.q, nl = m.nloc();
  int nq = (d == 2) ? q * q : q * q * q;
  if (!dg) std::fill(b, b + m.ndof, 0.0); else std::fill(b, b + m.nel * nl, 0.0);
  for (i64 e = 0; e < m.nel; ++e)
    for (int iq = 0; iq < nq; ++iq) {
      int qc[3] = {iq % q, (iq / q) % q, iq / (q * q)};
      double xi[3], x[3], J[9], Ji[9], w = 1.0;
      for (int k = 0; k < d; ++k) { xi[k] = m.b.xg[qc[k]]; w *= m.b.wg[qc[k]]; }
      m.map(e, xi, x, J);
      double det = det_inv(d, J, Ji);
      double f = fq[e * nq + iq] * w * det;
      for (int a = 0; a < nl; ++a) {
        int lc[3]; m.local_coords(a, lc);
        double phi = 1.0;
        for (int k = 0; k < d; ++k) phi *= m.b.B[qc[k] * (p + 1) + lc[k]];
        if (!dg) b[m.l2g(e, a)] += f * phi; else b[e * nl + a] += f * phi;
      }
    }
  if (!dg) for (i64 g = 0; g < m.ndof; ++g) if (m.is_dirichlet(g)) b[g] = 0.0;
  return 0;
}

// L2 error of a CG (dg=0) or DG (dg=1) nodal field against exact values at the quad points.
extern "C" double or_l2_error(void* h, const double* u, const double* uq, int dg) {
  Problem* P = (Problem*)h; const Mesh& m = P->m; const int d = m.d, p = m.p, q = m.b.q, nl = m.nloc();
  int nq = (d == 2) ? q * q : q * q * q;
  double s = 0.0;
  for (i64 e = 0; e < m.nel; ++e)
    for (int iq = 0; iq < nq; ++iq) {
      int qc[3] = {iq % q, (iq / q) % q, iq / (q * q)};
      double xi[3], x[3], J[9], Ji[9], w = 1.0;
      for (int k = 0; k < d; ++k) { xi[k] = m.b.xg[qc[k]]; w *= m.b.wg[qc[k]]; }
      m.map(e, xi, x, J);
      double det = det_inv(d, J, Ji);
      double uh = 0.0;
      for (int a = 0; a < nl; ++a) {
        int lc[3]; m.local_coords(a, lc);
        double phi = 1.0;
        for (int k = 0; k < d; ++k) phi *= m.b.B[qc[k] * (p + 1) + lc[k]];
        uh += phi * (dg ? u[e * nl + a] : u[m.l2g(e, a)]);
      }
      double err = uh - uq[e * nq + iq];
      s += w * det * err * err;
    }
  return std::sqrt(s);
}

// -----------------------------------------------------------------------------
// 8. Low-order-refined stiffness K_h: Q1 on every GLL subcell, the
//    subcell map being the element map restricted (= multilinear in the
//    subcell's corner images, reading c2), 2^d Gauss points per subcell.
//    Assembled on the full node grid (no Dirichlet elimination; the patch and
//    coarse spaces only ever use interior nodes).
// -----------------------------------------------------------------------------
static bool assemble_Kh(const Mesh& m, CSR& K) {
  const int d = m.d, p = m.p;
  const double g0 = 0.5 - 0.5 / std::sqrt(3.0), g1 = 0.5 + 0.5 / std::sqrt(3.0);
  const double gp[2] = {g0, g1};
  int nsub = (d == 2) ? p * p : p * p * p;
  int nc = 1 << d;
  std::vector<std::vector<Trip>> tl(m.nel);
  bool ok = true;
#pragma omp parallel for schedule(static)
  for (i64 e = 0; e < m.nel; ++e) {
    std::vector<Trip>& t = tl[e];
    for (int s = 0; s < nsub; ++s) {
      int sc[3] = {s % p, (s / p) % p, (d == 3) ? s / (p * p) : 0};
      // corner images of the GLL grid under the element map
      double X[8][3]; i64 gid[8];
      for (int c = 0; c < nc; ++c) {
        int cb[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
        double xi[3], x[3], J[9];
        int lc[3] = {0, 0, 0};
        for (int k = 0; k < d; ++k) { lc[k] = sc[k] + cb[k]; xi[k] = m.b.xi[lc[k]]; }
        m.map(e, xi, x, J);
        for (int k = 0; k < d; ++k) X[c][k] = x[k];
        int a = lc[0] + (p + 1) * (lc[1] + (p + 1) * lc[2]);
        gid[c] = m.l2g(e, a);
      }
      double Ks[8][8] = {{0}};
      int ngp = nc;
      for (int ig = 0; ig < ngp; ++ig) {
        int gb[3] = {ig & 1, (ig >> 1) & 1, (ig >> 2) & 1};
        double t3[3];
        for (int k = 0; k < d; ++k) t3[k] = gp[gb[k]];
        double J[9] = {0}, Ji[9], gr[8][3];
        for (int c = 0; c < nc; ++c) {
          int cb[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
          for (int k = 0; k < d; ++k) {
            double g = cb[k] ? 1.0 : -1.0;
            for (int mm = 0; mm < d; ++mm) if (mm != k) g *= cb[mm] ? t3[mm] : 1.0 - t3[mm];
            gr[c][k] = g;
            for (int i = 0; i < d; ++i) J[i * d + k] += X[c][i] * g;
          }
        }
        double det = det_inv(d, J, Ji);
        if (!(det > 0.0)) ok = false;
        double w = (d == 2) ? 0.25 : 0.125;
        if (!m.bs.empty()) {   // b sampled at the subcell Gauss point (SPEC S:233 reading)
          int ec[3], sg[3] = {0, 0, 0};
          m.elem_coords(e, ec);
          for (int k = 0; k < d; ++k) sg[k] = ec[k] * p + sc[k];
          w *= m.bs[(size_t)m.sub_index(sg) * nc + ig];
        }
        double pg[8][3];
        for (int c = 0; c < nc; ++c)
          for (int i = 0; i < d; ++i) {
            double v = 0.0;
            for (int k = 0; k < d; ++k) v += Ji[k * d + i] * gr[c][k];
            pg[c][i] = v;
          }
        for (int a = 0; a < nc; ++a)
          for (int bb = 0; bb < nc; ++bb) {
            double v = 0.0;
            for (int i = 0; i < d; ++i) v += pg[a][i] * pg[bb][i];
            Ks[a][bb] += w * det * v;
          }
      }
      for (int a = 0; a < nc; ++a)
        for (int bb = 0; bb < nc; ++bb) t.push_back({gid[a], (int)gid[bb], Ks[a][bb]});
    }
  }
  if (!ok) { g_err = "lor: degenerate subcell"; return false; }
  std::vector<Trip> all;
  for (auto& t : tl) { all.insert(all.end(), t.begin(), t.end()); std::vector<Trip>().swap(t); }
  K = csr_from_triplets(m.ndof, m.ndof, all);
  return true;
}

// Element-structured coarsening chain (reading c3): keep the end
// points, delete interior nodes at odd 1-based interior positions, until no
// interior node is left.
static std::vector<std::vector<int>> coarsening_chain(int p) {
  std::vector<std::vector<int>> ch;
  std::vector<int> cur;
  for (int i = 0; i <= p; ++i) cur.push_back(i);
  ch.push_back(cur);
  while (cur.size() > 2) {
    std::vector<int> nx;
    nx.push_back(cur.front());
    for (size_t t = 1; t + 1 < cur.size(); ++t)
      if (t % 2 == 0) nx.push_back(cur[t]);
    nx.push_back(cur.back());
    cur = nx; ch.push_back(cur);
  }
  return ch;
}

extern "C" int or_chain(int p, int* out, int* lens) {
  auto ch = coarsening_chain(p);
  int o = 0;
  for (size_t l = 0; l < ch.size(); ++l) {
    lens[l] = (int)ch[l].size();
    for (int v : ch[l]) out[o++] = v;
  }
  return (int)ch.size();
}

// 1D prolongation between consecutive chain levels on n elements: linear
// interpolation in the GLL reference coordinate within each element.
static CSR prolong_1d(const vec& xi, const std::vector<int>& fine, const std::vector<int>& coarse, int n) {
  int mf = (int)fine.size(), mc = (int)coarse.size();
  i64 Nf = (i64)n * (mf - 1) + 1, Nc = (i64)n * (mc - 1) + 1;
  std::vector<Trip> t;
  for (int e = 0; e < n; ++e)
    for (int tf = 0; tf < mf; ++tf) {
      if (e > 0 && tf == 0) continue;  // shared node already emitted
      i64 gf = (i64)e * (mf - 1) + tf;
      int a = fine[tf];
      int hit = -1;
      for (int tc = 0; tc < mc; ++tc) if (coarse[tc] == a) hit = tc;
      if (hit >= 0) { t.push_back({gf, (int)(e * (mc - 1) + hit), 1.0}); continue; }
      int tl = 0;
      while (!(coarse[tl] < a && a < coarse[tl + 1])) ++tl;
      double xl = xi[coarse[tl]], xh = xi[coarse[tl + 1]], xa = xi[a];
      t.push_back({gf, (int)(e * (mc - 1) + tl), (xh - xa) / (xh - xl)});
      t.push_back({gf, (int)(e * (mc - 1) + tl + 1), (xa - xl) / (xh - xl)});
    }
  return csr_from_triplets(Nf, Nc, t);
}

// Kronecker product P = Pz (x) Py (x) Px on x-fastest grids.
static CSR kron3(const CSR& Px, const CSR& Py, const CSR* Pz) {
  std::vector<Trip> t;
  i64 nfx = Px.nr, nfy = Py.nr, ncx = Px.nc, ncy = Py.nc;
  i64 nfz = Pz ? Pz->nr : 1, ncz = Pz ? Pz->nc : 1;
  for (i64 k = 0; k < nfz; ++k)
    for (i64 j = 0; j < nfy; ++j)
      for (i64 i = 0; i < nfx; ++i) {
        i64 row = i + nfx * (j + nfy * k);
        i64 kb = Pz ? Pz->rp[k] : 0, ke = Pz ? Pz->rp[k + 1] : 1;
        for (i64 a = kb; a < ke; ++a)
          for (i64 b = Py.rp[j]; b < Py.rp[j + 1]; ++b)
            for (i64 c = Px.rp[i]; c < Px.rp[i + 1]; ++c) {
              i64 cz = Pz ? Pz->ci[a] : 0; double wz = Pz ? Pz->v[a] : 1.0;
              i64 col = Px.ci[c] + ncx * (Py.ci[b] + ncy * cz);
              t.push_back({row, (int)col, wz * Py.v[b] * Px.v[c]});
            }
      }
  return csr_from_triplets(nfx * nfy * nfz, ncx * ncy * ncz, t);
}

extern "C" int or_lor_assemble(void* h) {
  Problem* P = (Problem*)h; Mesh& m = P->m;
  if (P->lor_built) return 0;
  P->chain = coarsening_chain(m.p);
  P->Al.clear(); P->Pl.clear(); P->Nl.clear();
  CSR K;
  if (!assemble_Kh(m, K)) return 1;
  P->Al.push_back(K);
  for (auto& c : P->chain) P->Nl.push_back((int)c.size());
  for (size_t l = 0; l + 1 < P->chain.size(); ++l) {
    CSR px = prolong_1d(m.b.xi, P->chain[l], P->chain[l + 1], m.n[0]);
    CSR py = prolong_1d(m.b.xi, P->chain[l], P->chain[l + 1], m.n[1]);
    CSR pz;
    if (m.d == 3) pz = prolong_1d(m.b.xi, P->chain[l], P->chain[l + 1], m.n[2]);
    CSR Pf = kron3(px, py, m.d == 3 ? &pz : nullptr);
    P->Pl.push_back(Pf);
    P->Al.push_back(galerkin(P->Al[l], Pf));
  }
  P->lor_built = true;
  return 0;
}

// Export K_h (level l operator) in CSR form for tests.
extern "C" i64 or_level_nnz(void* h, int l) { return ((Problem*)h)->Al[l].nnz(); }
extern "C" i64 or_level_n(void* h, int l) { return ((Problem*)h)->Al[l].nr; }
extern "C" void or_level_csr(void* h, int l, i64* rp, int* ci, double* v) {
  const CSR& A = ((Problem*)h)->Al[l];
  std::copy(A.rp.begin(), A.rp.end(), rp);
  std::copy(A.ci.begin(), A.ci.end(), ci);
  std::copy(A.v.begin(), A.v.end(), v);
}
extern "C" int or_nlevels(void* h) { return (int)((Problem*)h)->chain.size(); }

// -----------------------------------------------------------------------------
// 9. MDF ordering fused with the ILU(0) elimination (readings c5/c6).
//    Current matrix At on the fixed pattern of A.  Discarded-fill weight of node
//    k: w_k^2 = sum over ordered pairs i != j of alive neighbours of k whose
//    entry (i,j) is not in the pattern of (At_ik At_kj / At_kk)^2.  Pick the
//    minimum of (q30(w^2), natural index); eliminate with the ILU(0) update on
//    the pattern only:  At_ij -= (At_ik At_kj) / At_kk  for alive i, j in N(k).
//    L_ik = At_ik / At_kk, D_k = At_kk.  M = L D L^T (reading c5).
// -----------------------------------------------------------------------------
static double q30(double x) {
  if (x == 0.0) return 0.0;
  int e; double f = std::frexp(x, &e);
  return std::ldexp(std::nearbyint(std::ldexp(f, 30)), e - 30);
}

static int find_in_row(const CSR& A, int i, int j) {
  auto b = A.ci.begin() + A.rp[i], e = A.ci.begin() + A.rp[i + 1];
  auto it = std::lower_bound(b, e, j);
  if (it != e && *it == j) return (int)(it - A.ci.begin());
  return -1;
}

static double mdf_weight2(const CSR& A, const vec& At, const std::vector<char>& alive, int k) {
  int kk = find_in_row(A, k, k);
  double akk = At[kk], s = 0.0;
  for (i64 a = A.rp[k]; a < A.rp[k + 1]; ++a) {
    int i = A.ci[a];
    if (i == k || !alive[i]) continue;
    for (i64 b = A.rp[k]; b < A.rp[k + 1]; ++b) {
      int j = A.ci[b];
      if (j == k || j == i || !alive[j]) continue;
      if (find_in_row(A, i, j) >= 0) continue;
      double f = (At[a] * At[b]) / akk;
      s += f * f;
    }
  }
  return s;
}

// Reverse Cuthill-McKee on the sparsity graph of A (P:599 cites it; definition and
// ties are reading r5): start at a node of minimum degree (lowest index
// among ties), breadth-first, each node's unvisited neighbours appended in order of
// (degree, index), restart at the next minimum-degree node if the graph is not
// connected; the elimination order is the reverse of the visiting order.
static std::vector<int> rcm_order(const CSR& A) {
  const int n = (int)A.nr;
  std::vector<int> deg(n, 0), seq, nb;
  std::vector<char> seen(n, 0);
  for (int i = 0; i < n; ++i)
    for (i64 a = A.rp[i]; a < A.rp[i + 1]; ++a) if (A.ci[a] != i) ++deg[i];
  while ((int)seq.size() < n) {
    int s = -1;
    for (int i = 0; i < n; ++i) if (!seen[i] && (s < 0 || deg[i] < deg[s])) s = i;
    seen[s] = 1;
    size_t head = seq.size();
    seq.push_back(s);
    while (head < seq.size()) {
      const int v = seq[head++];
      nb.clear();
      for (i64 a = A.rp[v]; a < A.rp[v + 1]; ++a) {
        const int u = A.ci[a];
        if (u != v && !seen[u]) { seen[u] = 1; nb.push_back(u); }
      }
      std::sort(nb.begin(), nb.end(), [&](int x, int y) { return deg[x] < deg[y] || (deg[x] == deg[y] && x < y); });
      seq.insert(seq.end(), nb.begin(), nb.end());
    }
  }
  std::reverse(seq.begin(), seq.end());
  return seq;
}

static bool mdf_ilu(PatchLevel& L, int ordering) {
  const CSR& A = L.A; int n = L.n;
  vec At = A.v;
  std::vector<char> alive(n, 1);
  vec w2(n, 0.0);
  L.order.assign(n, -1); L.pos.assign(n, -1);
  L.Lv.assign(A.nnz(), 0.0); L.Dg.assign(n, 0.0);
  if (ordering == 0)
    for (int k = 0; k < n; ++k) w2[k] = mdf_weight2(A, At, alive, k);
  const std::vector<int> rcm = ordering == 2 ? rcm_order(A) : std::vector<int>();
  for (int step = 0; step < n; ++step) {
    int kbest = -1; double key = 0.0;
    if (ordering == 2) kbest = rcm[step];
    else
      for (int k = 0; k < n; ++k) {
        if (!alive[k]) continue;
        double kq = (ordering == 0) ? q30(w2[k]) : 0.0;
        if (kbest < 0 || kq < key) { kbest = k; key = kq; }
      }
    int k = kbest;
    L.order[step] = k; L.pos[k] = step;
    int kk = find_in_row(A, k, k);
    double akk = At[kk];
    if (!(akk > 0.0)) {
      g_err = "ilu: non-positive pivot at step " + std::to_string(step);
      return false;
    }
    L.Dg[k] = akk;
    // L_ik for alive neighbours i (stored in row i, column k)
    for (i64 a = A.rp[k]; a < A.rp[k + 1]; ++a) {
      int i = A.ci[a];
      if (i == k || !alive[i]) continue;
      int ik = find_in_row(A, i, k);
      L.Lv[ik] = At[ik] / akk;
    }
    // ILU(0) update on the pattern
    for (i64 a = A.rp[k]; a < A.rp[k + 1]; ++a) {
      int i = A.ci[a];
      if (i == k || !alive[i]) continue;
      for (i64 b = A.rp[k]; b < A.rp[k + 1]; ++b) {
        int j = A.ci[b];
        if (j == k || !alive[j]) continue;
        int ij = find_in_row(A, i, j);
        if (ij < 0) continue;
        At[ij] = At[ij] - (At[a] * At[b]) / akk;
      }
    }
    alive[k] = 0;
    if (ordering == 0)
      for (i64 a = A.rp[k]; a < A.rp[k + 1]; ++a) {
        int i = A.ci[a];
        if (i != k && alive[i]) w2[i] = mdf_weight2(A, At, alive, i);
      }
  }
  return true;
}

// z = M^{-1} r with M = L D L^T in the elimination order (one ILU(0) smoothing step).
static void ilu_apply(const PatchLevel& L, const double* r, double* z) {
  const CSR& A = L.A; int n = L.n;
  vec y(r, r + n);
  for (int t = 0; t < n; ++t) {
    int k = L.order[t];
    double s = y[k];
    for (i64 a = A.rp[k]; a < A.rp[k + 1]; ++a) {
      int j = A.ci[a];
      if (L.pos[j] < t) s -= L.Lv[a] * y[j];
    }
    y[k] = s;
  }
  for (int k = 0; k < n; ++k) y[k] = y[k] / L.Dg[k];
  for (int t = n - 1; t >= 0; --t) {
    int k = L.order[t];
    double s = y[k];
    for (i64 a = A.rp[k]; a < A.rp[k + 1]; ++a) {
      int i = A.ci[a];
      if (L.pos[i] > t) {
        int ik = find_in_row(A, i, k);
        s -= L.Lv[ik] * y[i];
      }
    }
    y[k] = s;
  }
  std::copy(y.begin(), y.end(), z);
}

// Standalone MDF/ILU on a user CSR matrix (for the pins: tridiagonal, 3x3 Laplacian).
extern "C" int or_mdf_ilu_csr(int n, const i64* rp, const int* ci, const double* v, int ordering,
                              int* order_out, double* r, double* z) {
  PatchLevel L; L.n = n;
  L.A.nr = n; L.A.nc = n;
  L.A.rp.assign(rp, rp + n + 1);
  L.A.ci.assign(ci, ci + rp[n]);
  L.A.v.assign(v, v + rp[n]);
  if (!mdf_ilu(L, ordering)) return 1;
  std::copy(L.order.begin(), L.order.end(), order_out);
  if (r && z) ilu_apply(L, r, z);
  return 0;
}

// -----------------------------------------------------------------------------
// 10. Patches (eq:patch P:302-315) and their element-structured hierarchies.
// -----------------------------------------------------------------------------
// Level-l free-node box of a patch: element range [elo, ehi] per axis;
// nodes per element m_l = |chain[l]|; box [elo (m-1), (ehi+1)(m-1)], free =
// strict interior (homogeneous Dirichlet on the patch boundary).
static void patch_free_nodes(const Problem* P, const Patch& pt, int l, std::vector<i64>& gid) {
  const Mesh& m = P->m; int ml = P->Nl[l];
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, Ng[3] = {1, 1, 1};
  for (int k = 0; k < m.d; ++k) {
    lo[k] = pt.elo[k] * (ml - 1) + 1; hi[k] = (pt.ehi[k] + 1) * (ml - 1) - 1;
    Ng[k] = m.n[k] * (ml - 1) + 1;
  }
  gid.clear();
  for (int z = lo[2]; z <= hi[2]; ++z)
    for (int y = lo[1]; y <= hi[1]; ++y)
      for (int x = lo[0]; x <= hi[0]; ++x)
        gid.push_back(x + (i64)Ng[0] * (y + (i64)Ng[1] * z));
}

// Patch extension for isotropic overlap (sec:aniso P:1123-1128, "patches containing
// anisotropic elements are extended to ensure that the overlap remains isotropic";
// rule = reading r6): along each axis, with H the largest extent of the vertex
// patch's own elements on the vertex line through x_j, a side of the patch whose
// physical extent from x_j is below H / 2 grows by one element layer at a time
// (at most 4 elements per axis).
static void extend_vertex_patch(const Mesh& m, const int* vc, Patch& pt) {
  for (int k = 0; k < m.d; ++k) {
    auto xk = [&](int i) {
      int g[3] = {vc[0], vc[1], vc[2]};
      g[k] = i;
      const i64 vid = g[0] + (i64)m.nvx[0] * (g[1] + (i64)m.nvx[1] * g[2]);
      return m.V[(size_t)vid * m.d + k];
    };
    int lo = pt.elo[k], hi = pt.ehi[k];
    double H = 0.0;
    for (int i = lo; i <= hi; ++i) H = std::max(H, xk(i + 1) - xk(i));
    if (vc[k] > 0)
      while (xk(vc[k]) - xk(lo) < 0.5 * H && lo > 0 && hi - lo + 1 < 4) --lo;
    if (vc[k] < m.n[k])
      while (xk(hi + 1) - xk(vc[k]) < 0.5 * H && hi < m.n[k] - 1 && hi - lo + 1 < 4) ++hi;
    pt.elo[k] = lo; pt.ehi[k] = hi;
  }
}

static void make_patches(Problem* P) {
  const Mesh& m = P->m;
  P->patches.clear();
  if (P->patch_kind == 0) {  // one patch per vertex, E_j = {x_j}, all vertices
    for (i64 v = 0; v < m.nvert; ++v) {
      int vc[3] = {(int)(v % m.nvx[0]), (int)((v / m.nvx[0]) % m.nvx[1]), (int)(v / ((i64)m.nvx[0] * m.nvx[1]))};
      Patch pt;
      for (int k = 0; k < 3; ++k) {
        if (k >= m.d) { pt.elo[k] = pt.ehi[k] = 0; continue; }
        pt.elo[k] = std::max(vc[k] - 1, 0); pt.ehi[k] = std::min(vc[k], m.n[k] - 1);
      }
      if (P->extend) extend_vertex_patch(m, vc, pt);
      P->patches.push_back(pt);
    }
  } else if (P->patch_kind == 2) {  // single patch E_1 = all vertices, Omega_1 = Omega
    Patch pt;
    for (int k = 0; k < 3; ++k) { pt.elo[k] = 0; pt.ehi[k] = (k < m.d) ? m.n[k] - 1 : 0; }
    P->patches.push_back(pt);
  } else {  // element star: D_j and every element touching it (reading c9)
    for (i64 e = 0; e < m.nel; ++e) {
      int ec[3]; m.elem_coords(e, ec);
      Patch pt;
      for (int k = 0; k < 3; ++k) {
        if (k >= m.d) { pt.elo[k] = pt.ehi[k] = 0; continue; }
        pt.elo[k] = std::max(ec[k] - 1, 0); pt.ehi[k] = std::min(ec[k] + 1, m.n[k] - 1);
      }
      P->patches.push_back(pt);
    }
  }
}

// -----------------------------------------------------------------------------
// 11. Coarse space V_0 = Q1 on T_p and R_0 = GMG V(1,1) with
//     l1-Jacobi, 2:1 vertex-centred multilinear transfer, Galerkin, coarsest
//     exact (reading c11, replacing BoomerAMG).
// -----------------------------------------------------------------------------
static CSR vertex_prolongation(const Mesh& m) {
  // P_0: vertex value -> LOR node value, multilinear in the reference coordinate
  std::vector<CSR> P1(3);
  for (int k = 0; k < m.d; ++k) {
    std::vector<Trip> t;
    for (int e = 0; e < m.n[k]; ++e)
      for (int a = 0; a <= m.p; ++a) {
        if (e > 0 && a == 0) continue;
        i64 g = (i64)e * m.p + a;
        double x = m.b.xi[a];
        if (a == 0) t.push_back({g, e, 1.0});
        else if (a == m.p) t.push_back({g, e + 1, 1.0});
        else { t.push_back({g, e, 1.0 - x}); t.push_back({g, e + 1, x}); }
      }
    P1[k] = csr_from_triplets((i64)m.n[k] * m.p + 1, m.n[k] + 1, t);
  }
  return kron3(P1[0], P1[1], m.d == 3 ? &P1[2] : nullptr);
}

static std::vector<i64> interior_ids(int d, const int* nv) {
  std::vector<i64> ids;
  int nz = (d == 3) ? nv[2] : 1;
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < nv[1]; ++y)
      for (int x = 0; x < nv[0]; ++x) {
        bool in = x > 0 && x < nv[0] - 1 && y > 0 && y < nv[1] - 1 && (d == 2 || (z > 0 && z < nz - 1));
        if (in) ids.push_back(x + (i64)nv[0] * (y + (i64)nv[1] * z));
      }
  return ids;
}

// 2:1 vertex-centred 1D interpolation, n coarse intervals -> 2n fine intervals
static CSR gmg_prolong_1d(int nc) {
  std::vector<Trip> t;
  for (int f = 0; f <= 2 * nc; ++f) {
    if (f % 2 == 0) t.push_back({f, f / 2, 1.0});
    else { t.push_back({f, f / 2, 0.5}); t.push_back({f, f / 2 + 1, 0.5}); }
  }
  return csr_from_triplets(2 * nc + 1, nc + 1, t);
}

static bool build_coarse(Problem* P) {
  const Mesh& m = P->m;
  P->P0 = vertex_prolongation(m);
  int nv[3] = {m.nvx[0], m.nvx[1], m.nvx[2]};
  P->cfree = interior_ids(m.d, nv);
  CSR A0full = galerkin(P->Al[0], P->P0);
  CSR A0 = csr_submatrix(A0full, P->cfree, P->cfree);
  P->Ac.clear(); P->Pc.clear(); P->dl1.clear(); P->cn.clear();
  if (P->coarse == 2) {  // exact coarse solve (test configuration)
    int n = (int)A0.nr;
    P->C0dense.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i)
      for (i64 k = A0.rp[i]; k < A0.rp[i + 1]; ++k) P->C0dense[(size_t)i * n + A0.ci[k]] = A0.v[k];
    P->n0dense = n;
    if (n > 0 && !cholesky(n, P->C0dense)) { g_err = "coarse: A_0 not SPD"; return false; }
    return true;
  }
  P->Ac.push_back(A0);
  std::vector<int> cur(nv, nv + 3);
  P->cn.push_back(cur);
  // coarsen while every used axis has an even number (>2) of intervals
  while (true) {
    bool can = true;
    for (int k = 0; k < m.d; ++k) if ((cur[k] - 1) % 2 != 0 || cur[k] - 1 <= 2) can = false;
    if (!can) break;
    std::vector<int> nxt = cur;
    for (int k = 0; k < m.d; ++k) nxt[k] = (cur[k] - 1) / 2 + 1;
    CSR px = gmg_prolong_1d(nxt[0] - 1), py = gmg_prolong_1d(nxt[1] - 1), pz;
    if (m.d == 3) pz = gmg_prolong_1d(nxt[2] - 1);
    CSR Pfull = kron3(px, py, m.d == 3 ? &pz : nullptr);
    std::vector<i64> fi = interior_ids(m.d, cur.data()), ci = interior_ids(m.d, nxt.data());
    CSR Pi = csr_submatrix(Pfull, fi, ci);
    P->Pc.push_back(Pi);
    P->Ac.push_back(galerkin(P->Ac.back(), Pi));
    P->cn.push_back(nxt);
    cur = nxt;
  }
  for (auto& A : P->Ac) {
    vec dd(A.nr, 0.0);
    for (i64 i = 0; i < A.nr; ++i)
      for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) dd[i] += std::fabs(A.v[k]);
    P->dl1.push_back(dd);
  }
  const CSR& Al = P->Ac.back();
  P->ncc = (int)Al.nr;
  P->Cc.assign((size_t)P->ncc * P->ncc, 0.0);
  for (int i = 0; i < P->ncc; ++i)
    for (i64 k = Al.rp[i]; k < Al.rp[i + 1]; ++k) P->Cc[(size_t)i * P->ncc + Al.ci[k]] = Al.v[k];
  if (P->ncc > 0 && !cholesky(P->ncc, P->Cc)) { g_err = "coarse: coarsest not SPD"; return false; }
  return true;
}

// One GMG V(1,1) cycle with l1-Jacobi smoothing, zero initial guess.
static void gmg_vcycle(const Problem* P, size_t l, const vec& r, vec& z) {
  const CSR& A = P->Ac[l];
  i64 n = A.nr;
  z.assign(n, 0.0);
  if (l + 1 == P->Ac.size()) {
    z = r;
    if (n > 0) chol_solve((int)n, P->Cc, z.data());
    return;
  }
  const vec& dd = P->dl1[l];
  for (i64 i = 0; i < n; ++i) z[i] = r[i] / dd[i];          // pre-smoothing
  vec Az(n), s(n);
  A.matvec(z.data(), Az.data());
  for (i64 i = 0; i < n; ++i) s[i] = r[i] - Az[i];
  const CSR& Pc = P->Pc[l];
  vec rc(Pc.nc, 0.0);
  for (i64 i = 0; i < Pc.nr; ++i)                             // restriction P^T s
    for (i64 k = Pc.rp[i]; k < Pc.rp[i + 1]; ++k) rc[Pc.ci[k]] += Pc.v[k] * s[i];
  vec ec;
  gmg_vcycle(P, l + 1, rc, ec);
  for (i64 i = 0; i < Pc.nr; ++i)                             // prolongation
    for (i64 k = Pc.rp[i]; k < Pc.rp[i + 1]; ++k) z[i] += Pc.v[k] * ec[Pc.ci[k]];
  A.matvec(z.data(), Az.data());
  for (i64 i = 0; i < n; ++i) z[i] += (r[i] - Az[i]) / dd[i]; // post-smoothing
}

// -----------------------------------------------------------------------------
// 12. Schwarz setup / apply
// -----------------------------------------------------------------------------
extern "C" int or_schwarz_setup2(void* h, int patch_kind, int ordering, int coarse, int local_exact) {
  Problem* P = (Problem*)h;
  if (or_lor_assemble(h)) return 1;
  P->patch_kind = patch_kind; P->ordering = ordering; P->coarse = coarse; P->local_exact = local_exact;
  make_patches(P);
  const int L = local_exact ? 1 : (int)P->chain.size();
  bool ok = true;
  std::string err;
#pragma omp parallel for schedule(dynamic, 4)
  for (i64 j = 0; j < (i64)P->patches.size(); ++j) {
    Patch& pt = P->patches[j];
    pt.lv.assign(L, PatchLevel());
    for (int l = 0; l < L; ++l) {
      PatchLevel& lv = pt.lv[l];
      patch_free_nodes(P, pt, l, lv.gid);
      lv.n = (int)lv.gid.size();
      lv.A = csr_submatrix(P->Al[l], lv.gid, lv.gid);
      lv.coarsest = (l == L - 1);
      if (l > 0) pt.lv[l - 1].P = csr_submatrix(P->Pl[l - 1], pt.lv[l - 1].gid, lv.gid);
      if (lv.coarsest) {
        lv.C.assign((size_t)lv.n * lv.n, 0.0);
        for (int i = 0; i < lv.n; ++i)
          for (i64 k = lv.A.rp[i]; k < lv.A.rp[i + 1]; ++k) lv.C[(size_t)i * lv.n + lv.A.ci[k]] = lv.A.v[k];
        if (lv.n > 0 && !cholesky(lv.n, lv.C)) {
#pragma omp critical
          { ok = false; err = "patch " + std::to_string(j) + ": coarsest not SPD"; }
        }
      } else if (!mdf_ilu(lv, ordering)) {
#pragma omp critical
        { ok = false; err = "patch " + std::to_string(j) + " level " + std::to_string(l) + ": " + g_err; }
      }
    }
  }
  if (!ok) { g_err = err; return 1; }
  if (coarse != 1 && !build_coarse(P)) return 1;
  P->schwarz_built = true;
  return 0;
}
extern "C" int or_set_patch_extension(void* h, int extend) {
  ((Problem*)h)->extend = extend ? 1 : 0;
  return 0;
}
extern "C" int or_patch_range(void* h, i64 j, int* elo, int* ehi) {
  const Problem* P = (const Problem*)h;
  if (j < 0 || j >= (i64)P->patches.size()) { g_err = "patch index"; return 1; }
  for (int k = 0; k < 3; ++k) { elo[k] = P->patches[j].elo[k]; ehi[k] = P->patches[j].ehi[k]; }
  return 0;
}
extern "C" int or_schwarz_setup(void* h, int patch_kind, int ordering, int coarse) {
  return or_schwarz_setup2(h, patch_kind, ordering, coarse, 0);
}

extern "C" i64 or_npatches(void* h) { return (i64)((Problem*)h)->patches.size(); }
extern "C" int or_patch_level_n(void* h, i64 j, int l) { return ((Problem*)h)->patches[j].lv[l].n; }
extern "C" void or_patch_ordering(void* h, i64 j, int l, int* order) {
  const PatchLevel& lv = ((Problem*)h)->patches[j].lv[l];
  std::copy(lv.order.begin(), lv.order.end(), order);
}

// Patch V(1,1) cycle, zero initial guess, recursive over levels.
static void gmg_vcycle(const Problem* P, size_t l, const vec& r, vec& z);
// B(1): the single patch's V-cycle has the coarse solve at its bottom —
// its coarsest level is the p = 1 problem on T_p, solved by R_0 (one GMG V-cycle,
// reading c11; coarse = 2: exactly) instead of the dense factor of reading c8.
static void patch_vcycle(const Problem* P, const Patch& pt, int l, const vec& r, vec& z) {
  const PatchLevel& L = pt.lv[l];
  int n = L.n;
  z.assign(n, 0.0);
  if (n == 0) return;
  if (L.coarsest) {
    if (P->patch_kind == 2 && P->coarse == 0) { gmg_vcycle(P, 0, r, z); return; }
    if (P->patch_kind == 2 && P->coarse == 2) { z = r; if (P->n0dense) chol_solve(P->n0dense, P->C0dense, z.data()); return; }
    z = r; chol_solve(n, L.C, z.data()); return;
  }
  ilu_apply(L, r.data(), z.data());                          // pre-smoothing
  vec Az(n), s(n);
  L.A.matvec(z.data(), Az.data());
  for (int i = 0; i < n; ++i) s[i] = r[i] - Az[i];
  const CSR& Pm = L.P;
  vec rc(Pm.nc, 0.0);
  for (i64 i = 0; i < Pm.nr; ++i)
    for (i64 k = Pm.rp[i]; k < Pm.rp[i + 1]; ++k) rc[Pm.ci[k]] += Pm.v[k] * s[i];
  vec ec;
  patch_vcycle(P, pt, l + 1, rc, ec);
  for (i64 i = 0; i < Pm.nr; ++i)
    for (i64 k = Pm.rp[i]; k < Pm.rp[i + 1]; ++k) z[i] += Pm.v[k] * ec[Pm.ci[k]];
  L.A.matvec(z.data(), Az.data());
  for (int i = 0; i < n; ++i) s[i] = r[i] - Az[i];
  vec w(n);
  ilu_apply(L, s.data(), w.data());                          // post-smoothing
  for (int i = 0; i < n; ++i) z[i] += w[i];
}

// z = B r = sum_j I_j R_j I_j^T r + P_0 R_0 P_0^T r  (eq:as), z_D = 0.
// `which`: 1 = patches only, 2 = coarse only, 3 = both.
static void schwarz_apply(const Problem* P, const double* r, double* z, int which) {
  const Mesh& m = P->m;
  std::fill(z, z + m.ndof, 0.0);
  if (which & 1) {
    std::vector<vec> zj(P->patches.size());
#pragma omp parallel for schedule(dynamic, 16)
    for (i64 j = 0; j < (i64)P->patches.size(); ++j) {
      const Patch& pt = P->patches[j];
      const PatchLevel& L0 = pt.lv[0];
      vec rj(L0.n);
      for (int i = 0; i < L0.n; ++i) rj[i] = r[L0.gid[i]];
      patch_vcycle(P, pt, 0, rj, zj[j]);
    }
    for (size_t j = 0; j < P->patches.size(); ++j) {        // fixed order (a8)
      const PatchLevel& L0 = P->patches[j].lv[0];
      for (int i = 0; i < L0.n; ++i) z[L0.gid[i]] += zj[j][i];
    }
  }
  if ((which & 2) && P->coarse != 1 && P->patch_kind != 2) {  // B(1): R_0 sits inside the V-cycle
    const CSR& P0 = P->P0;
    vec rcf(P0.nc, 0.0);
    for (i64 i = 0; i < P0.nr; ++i)
      for (i64 k = P0.rp[i]; k < P0.rp[i + 1]; ++k) rcf[P0.ci[k]] += P0.v[k] * r[i];
    vec rc(P->cfree.size());
    for (size_t i = 0; i < P->cfree.size(); ++i) rc[i] = rcf[P->cfree[i]];
    vec zc;
    if (P->coarse == 2) { zc = rc; if (P->n0dense) chol_solve(P->n0dense, P->C0dense, zc.data()); }
    else gmg_vcycle(P, 0, rc, zc);
    vec zcf(P0.nc, 0.0);
    for (size_t i = 0; i < P->cfree.size(); ++i) zcf[P->cfree[i]] = zc[i];
    for (i64 i = 0; i < P0.nr; ++i) {
      double s = 0.0;
      for (i64 k = P0.rp[i]; k < P0.rp[i + 1]; ++k) s += P0.v[k] * zcf[P0.ci[k]];
      z[i] += s;
    }
  }
  for (i64 g = 0; g < m.ndof; ++g) if (m.is_dirichlet(g)) z[g] = 0.0;
}

// -----------------------------------------------------------------------------
// 13. SIPG operator (eq:ip P:113-136) and the DG preconditioner (eq:dg-as).
// -----------------------------------------------------------------------------
void dg_apply(const Problem* P, const double* x, double* y);
static void dg_precond(const Problem* P, const double* r, double* z);

// -----------------------------------------------------------------------------
// 14. Public operator / preconditioner entry points
// -----------------------------------------------------------------------------
extern "C" int or_apply_K(void* h, const double* x, double* y) {
  Problem* P = (Problem*)h;
  if (P->disc == 0) {
    if (!P->cached && P->m.nel * (i64)P->m.nloc() * P->m.nloc() <= (i64)1 << 30) build_elem_cache(P);
    cg_apply(P, x, y);
  } else {
    dg_apply(P, x, y);
  }
  return 0;
}

extern "C" int or_precond_apply(void* h, const double* r, double* z, int which) {
  Problem* P = (Problem*)h;
  if (!P->schwarz_built) { g_err = "schwarz not built"; return 1; }
  if (P->disc == 0) schwarz_apply(P, r, z, which);
  else dg_precond(P, r, z);
  return 0;
}

// -----------------------------------------------------------------------------
// 15. Preconditioned conjugate gradients (reading c12):
//     x0 = 0, stop when ||r_k||_2 <= tol ||b||_2 (recursively updated residual).
// -----------------------------------------------------------------------------
static double dot(i64 n, const double* a, const double* b) {
  double s = 0.0;
  for (i64 i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

extern "C" int or_pcg(void* h, const double* b, double* x, double tol, int maxit, int* iters,
                      double* res_hist, double* alpha, double* beta) {
  Problem* P = (Problem*)h;
  i64 n = (P->disc == 0) ? P->m.ndof : P->m.nel * P->m.nloc();
  vec r(b, b + n), z(n), p(n), q(n);
  std::fill(x, x + n, 0.0);
  double nb = std::sqrt(dot(n, b, b));
  res_hist[0] = 1.0;
  *iters = 0;
  if (nb == 0.0) return 0;
  or_precond_apply(h, r.data(), z.data(), 3);
  p = z;
  double rho = dot(n, r.data(), z.data());
  for (int k = 1; k <= maxit; ++k) {
    or_apply_K(h, p.data(), q.data());
    double pq = dot(n, p.data(), q.data());
    if (!(pq > 0.0)) { g_err = "pcg: breakdown p.Ap <= 0 at iteration " + std::to_string(k); *iters = k; return 2; }
    double a = rho / pq;
    alpha[k - 1] = a;
    for (i64 i = 0; i < n; ++i) { x[i] += a * p[i]; r[i] -= a * q[i]; }
    double nr = std::sqrt(dot(n, r.data(), r.data()));
    res_hist[k] = nr / nb;
    *iters = k;
    if (nr <= tol * nb) return 0;
    or_precond_apply(h, r.data(), z.data(), 3);
    double rho2 = dot(n, r.data(), z.data());
    if (!(rho2 > 0.0)) { g_err = "pcg: breakdown r.z <= 0 at iteration " + std::to_string(k); return 2; }
    double bb = rho2 / rho;
    beta[k - 1] = bb;
    rho = rho2;
    for (i64 i = 0; i < n; ++i) p[i] = z[i] + bb * p[i];
  }
  g_err = "pcg: not converged";
  return 3;
}

#include "lorpc_oracle_dg.inc"
