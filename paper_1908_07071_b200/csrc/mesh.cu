// Mesh geometry (row a1): geometric factors at Gauss points, node coordinates,
// element volumes, quadrature points and load vectors.
//
// G_q = w_q det J_q J_q^{-1} J_q^{-T} (symmetric, d(d+1)/2 components) at the
// q^d Gauss points (q = p+1, reading c1) of the multilinear element map
// (P:82-84).  Layout [n_el][ncomp][q^d] so a warp of quadrature-point threads
// reads each component with unit stride.
#include "device.cuh"

namespace lorpc {

template <int DIM>
__global__ void k_geom(const double* __restrict__ V, int3 n, Basis1D bs, double* __restrict__ G,
                       double* __restrict__ vol, unsigned long long* bad, const double* __restrict__ bq) {
  const int q = bs.q;
  const int nq = DIM == 2 ? q * q : q * q * q;
  const long long nel = (long long)n.x * n.y * (DIM == 3 ? n.z : 1);
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (tid >= nel * nq) return;
  const long long e = tid / nq;
  const int iq = (int)(tid % nq);
  const int ex = (int)(e % n.x), ey = (int)((e / n.x) % n.y), ez = DIM == 3 ? (int)(e / ((long long)n.x * n.y)) : 0;
  const int qc[3] = {iq % q, (iq / q) % q, iq / (q * q)};
  double xi[3], x[3], J[9], Ji[9];
  double w = 1.0;
#pragma unroll
  for (int k = 0; k < DIM; ++k) { xi[k] = bs.xq[qc[k]]; w *= bs.wq[qc[k]]; }
  const int nv[3] = {n.x + 1, n.y + 1, n.z + 1};
  elem_map<DIM>(V, nv, ex, ey, ez, xi, x, J);
  const double det = inv_det<DIM>(J, Ji);
  if (!(det > 0.0)) atomicMin(bad, (unsigned long long)e);
  // b(x_q) w_q det J_q J^{-1} J^{-T} (sec:variable-coeff; b = 1 unless set)
  const double f = w * det * (bq ? bq[tid] : 1.0);
  constexpr int NC = DIM == 2 ? 3 : 6;
  double* Ge = G + e * NC * nq;
  int c = 0;
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int j = i; j < DIM; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < DIM; ++k) s += Ji[i * DIM + k] * Ji[j * DIM + k];  // (J^{-1} J^{-T})_{ij}
      Ge[c * nq + iq] = f * s;
      ++c;
    }
  if (vol) atomicAdd(vol + e, w * det);
}

// Physical coordinates of the GLL nodes (images of the GLL grid under the
// element map).
template <int DIM>
__global__ void k_node_coords(const double* __restrict__ V, int3 n, int3 N, Basis1D bs, double* __restrict__ X) {
  const long long ndof = (long long)N.x * N.y * N.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= ndof) return;
  const int gc[3] = {(int)(g % N.x), (int)((g / N.x) % N.y), (int)(g / ((long long)N.x * N.y))};
  const int nn[3] = {n.x, n.y, n.z};
  int ec[3] = {0, 0, 0};
  double xi[3];
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    ec[k] = min(gc[k] / bs.p, nn[k] - 1);
    xi[k] = bs.xi[gc[k] - ec[k] * bs.p];
  }
  const int nv[3] = {n.x + 1, n.y + 1, n.z + 1};
  double x[3], J[9];
  elem_map<DIM>(V, nv, ec[0], ec[1], ec[2], xi, x, J);
#pragma unroll
  for (int k = 0; k < DIM; ++k) X[g * DIM + k] = x[k];
}

template <int DIM>
__global__ void k_quad_points(const double* __restrict__ V, int3 n, Basis1D bs, double* __restrict__ Xq) {
  const int q = bs.q;
  const int nq = DIM == 2 ? q * q : q * q * q;
  const long long nel = (long long)n.x * n.y * (DIM == 3 ? n.z : 1);
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (tid >= nel * nq) return;
  const long long e = tid / nq;
  const int iq = (int)(tid % nq);
  const int ex = (int)(e % n.x), ey = (int)((e / n.x) % n.y), ez = DIM == 3 ? (int)(e / ((long long)n.x * n.y)) : 0;
  const int qc[3] = {iq % q, (iq / q) % q, iq / (q * q)};
  double xi[3], x[3], J[9];
#pragma unroll
  for (int k = 0; k < DIM; ++k) xi[k] = bs.xq[qc[k]];
  const int nv[3] = {n.x + 1, n.y + 1, n.z + 1};
  elem_map<DIM>(V, nv, ex, ey, ez, xi, x, J);
#pragma unroll
  for (int k = 0; k < DIM; ++k) Xq[tid * DIM + k] = x[k];
}

// b_a = sum_q w_q det J_q f(x_q) phi_a(x_q): one thread per (element, node).
template <int DIM>
__global__ void k_rhs(const double* __restrict__ V, int3 n, int3 N, Basis1D bs, const double* __restrict__ fq,
                      double* __restrict__ b, int dg) {
  const int p = bs.p, q = bs.q;
  const int nl = DIM == 2 ? (p + 1) * (p + 1) : (p + 1) * (p + 1) * (p + 1);
  const int nq = DIM == 2 ? q * q : q * q * q;
  const long long nel = (long long)n.x * n.y * (DIM == 3 ? n.z : 1);
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (tid >= nel * nl) return;
  const long long e = tid / nl;
  const int a = (int)(tid % nl);
  const int ac[3] = {a % (p + 1), (a / (p + 1)) % (p + 1), a / ((p + 1) * (p + 1))};
  const int ex = (int)(e % n.x), ey = (int)((e / n.x) % n.y), ez = DIM == 3 ? (int)(e / ((long long)n.x * n.y)) : 0;
  const int nv[3] = {n.x + 1, n.y + 1, n.z + 1};
  double s = 0.0;
  for (int iq = 0; iq < nq; ++iq) {
    const int qc[3] = {iq % q, (iq / q) % q, iq / (q * q)};
    double xi[3], x[3], J[9], Ji[9], w = 1.0, phi = 1.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      xi[k] = bs.xq[qc[k]]; w *= bs.wq[qc[k]]; phi *= bs.B[qc[k] * (p + 1) + ac[k]];
    }
    elem_map<DIM>(V, nv, ex, ey, ez, xi, x, J);
    const double det = inv_det<DIM>(J, Ji);
    s += w * det * fq[e * nq + iq] * phi;
  }
  if (dg) {
    b[e * nl + a] = s;
  } else {
    const int g[3] = {ex * p + ac[0], ey * p + ac[1], DIM == 3 ? ez * p + ac[2] : 0};
    const long long gi = g[0] + (long long)N.x * (g[1] + (long long)N.y * g[2]);
    atomicAdd(b + gi, s);
  }
}

template <int DIM>
__global__ void k_zero_dirichlet(int3 N, double* __restrict__ b) {
  const long long ndof = (long long)N.x * N.y * N.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= ndof) return;
  const int gx = (int)(g % N.x), gy = (int)((g / N.x) % N.y), gz = (int)(g / ((long long)N.x * N.y));
  bool d = gx == 0 || gx == N.x - 1 || gy == 0 || gy == N.y - 1;
  if (DIM == 3) d = d || gz == 0 || gz == N.z - 1;
  if (d) b[g] = 0.0;
}

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

int geom_setup(lorpc_mesh* m, cudaStream_t s) {
  const int d = m->d;
  const int nc = d == 2 ? 3 : 6;
  if (!m->G) LORPC_TRY(dalloc(&m->G, (size_t)m->nel * nc * m->nq));
  if (!m->X) LORPC_TRY(dalloc(&m->X, (size_t)m->ndof_cg * d));
  if (!m->vol) LORPC_TRY(dalloc(&m->vol, (size_t)m->nel));
  LORPC_CUDA(cudaMemsetAsync(m->vol, 0, sizeof(double) * m->nel, s));
  unsigned long long* bad;
  LORPC_CUDA(cudaMallocHost(&bad, sizeof(unsigned long long)));
  unsigned long long* dbad;
  LORPC_TRY(dalloc(&dbad, 1));
  const unsigned long long init = ~0ull;
  LORPC_CUDA(cudaMemcpyAsync(dbad, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  long long tot = m->nel * m->nq;
  if (d == 2) k_geom<2><<<nblk(tot, 128), 128, 0, s>>>(m->V, n, m->basis, m->G, m->vol, dbad, m->bq);
  else k_geom<3><<<nblk(tot, 128), 128, 0, s>>>(m->V, n, m->basis, m->G, m->vol, dbad, m->bq);
  LORPC_LAUNCHED();
  if (d == 2) k_node_coords<2><<<nblk(m->ndof_cg, 256), 256, 0, s>>>(m->V, n, N, m->basis, m->X);
  else k_node_coords<3><<<nblk(m->ndof_cg, 256), 256, 0, s>>>(m->V, n, N, m->basis, m->X);
  LORPC_LAUNCHED();
  LORPC_CUDA(cudaMemcpyAsync(bad, dbad, sizeof(init), cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  unsigned long long e = *bad;
  cudaFreeHost(bad);
  dfree(dbad);
  if (e != ~0ull) return fail(LORPC_ERR_INVERTED_ELEMENT, "inverted element " + std::to_string(e));
  return LORPC_OK;
}

// Gauss points of the LOR subcells (reading c2: the subcell map is multilinear in
// the images of its corner GLL nodes; 2^d points t = 1/2 -+ 1/(2 sqrt 3)), global
// subcell index sx + (N0-1)(sy + (N1-1) sz) major, point bits x, y, z minor.
template <int DIM>
__global__ void k_subcell_points(const double* __restrict__ X, int3 N, double* __restrict__ Xs) {
  constexpr int NC = 1 << DIM;
  const long long ns = (long long)(N.x - 1) * (N.y - 1) * (DIM == 3 ? N.z - 1 : 1);
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= ns * NC) return;
  const long long sidx = t / NC;
  const int ig = (int)(t % NC);
  const int sc[3] = {(int)(sidx % (N.x - 1)), (int)((sidx / (N.x - 1)) % (N.y - 1)),
                     DIM == 3 ? (int)(sidx / ((long long)(N.x - 1) * (N.y - 1))) : 0};
  const double gp[2] = {0.5 - 0.5 / sqrt(3.0), 0.5 + 0.5 / sqrt(3.0)};
  double o[3] = {0.0, 0.0, 0.0};
  for (int c = 0; c < NC; ++c) {
    double wv = 1.0;
    long long id = 0, str = 1;
    const int Nn[3] = {N.x, N.y, N.z};
    for (int k = 0; k < DIM; ++k) {
      const int cb = (c >> k) & 1;
      const double tk = gp[(ig >> k) & 1];
      wv *= cb ? tk : 1.0 - tk;
      id += (sc[k] + cb) * str;
      str *= Nn[k];
    }
    for (int i = 0; i < DIM; ++i) o[i] += wv * X[id * DIM + i];
  }
  for (int i = 0; i < DIM; ++i) Xs[t * DIM + i] = o[i];
}

long long n_subcells(const lorpc_mesh* m) {
  long long n = 1;
  for (int k = 0; k < m->d; ++k) n *= m->N[k] - 1;
  return n;
}

int subcell_points(const lorpc_mesh* m, double* xs, cudaStream_t s) {
  const long long tot = n_subcells(m) << m->d;
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  if (m->d == 2) k_subcell_points<2><<<nblk(tot, 128), 128, 0, s>>>(m->X, N, xs);
  else k_subcell_points<3><<<nblk(tot, 128), 128, 0, s>>>(m->X, N, xs);
  LORPC_LAUNCHED();
  return LORPC_OK;
}

__global__ void k_min_positive(const double* __restrict__ v, long long n, int* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!(v[i] > 0.0)) *bad = 1;
}

// b at the volume Gauss points (K_p) and the LOR subcell Gauss points (K_h); copies
// them, re-forms G and checks b > 0
int set_coefficient(lorpc_mesh* m, const double* bq, const double* bs, cudaStream_t s) {
  const long long nqt = m->nel * m->nq, nst = n_subcells(m) << m->d;
  int* dbad = nullptr;
  LORPC_TRY(dalloc(&dbad, 1));
  LORPC_CUDA(cudaMemsetAsync(dbad, 0, sizeof(int), s));
  if (bq) {
    if (!m->bq) LORPC_TRY(dalloc(&m->bq, (size_t)nqt));
    LORPC_CUDA(cudaMemcpyAsync(m->bq, bq, sizeof(double) * nqt, cudaMemcpyDeviceToDevice, s));
    k_min_positive<<<296, 256, 0, s>>>(m->bq, nqt, dbad);
    LORPC_LAUNCHED();
  } else {
    dfree(m->bq);
  }
  if (bs) {
    if (!m->bsub) LORPC_TRY(dalloc(&m->bsub, (size_t)nst));
    LORPC_CUDA(cudaMemcpyAsync(m->bsub, bs, sizeof(double) * nst, cudaMemcpyDeviceToDevice, s));
    k_min_positive<<<296, 256, 0, s>>>(m->bsub, nst, dbad);
    LORPC_LAUNCHED();
  } else {
    dfree(m->bsub);
  }
  int bad = 0;
  LORPC_CUDA(cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  dfree(dbad);
  if (bad) { dfree(m->bq); dfree(m->bsub); return fail(LORPC_ERR_ARG, "set_coefficient: b must be > 0"); }
  return geom_setup(m, s);
}

int quad_points(const lorpc_mesh* m, double* xq, double* xbq, cudaStream_t s) {
  int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  if (xq) {
    long long tot = m->nel * m->nq;
    if (m->d == 2) k_quad_points<2><<<nblk(tot, 128), 128, 0, s>>>(m->V, n, m->basis, xq);
    else k_quad_points<3><<<nblk(tot, 128), 128, 0, s>>>(m->V, n, m->basis, xq);
    LORPC_LAUNCHED();
  }
  if (xbq) {
    extern int dg_bface_points(const lorpc_mesh* m, double* xbq, cudaStream_t s);
    LORPC_TRY(dg_bface_points(m, xbq, s));
  }
  return LORPC_OK;
}

int dg_rhs_bc(const lorpc_mesh* m, const double* gq, double* b, cudaStream_t s);

int rhs_assemble(const lorpc_mesh* m, const double* fq, const double* gq, double* b, cudaStream_t s) {
  int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  const int dg = m->desc.disc != 0;
  if (!dg) LORPC_CUDA(cudaMemsetAsync(b, 0, sizeof(double) * m->ndof, s));
  long long tot = m->nel * m->nloc;
  if (m->d == 2) k_rhs<2><<<nblk(tot, 128), 128, 0, s>>>(m->V, n, N, m->basis, fq, b, dg);
  else k_rhs<3><<<nblk(tot, 128), 128, 0, s>>>(m->V, n, N, m->basis, fq, b, dg);
  LORPC_LAUNCHED();
  if (!dg) {
    if (m->d == 2) k_zero_dirichlet<2><<<nblk(m->ndof, 256), 256, 0, s>>>(N, b);
    else k_zero_dirichlet<3><<<nblk(m->ndof, 256), 256, 0, s>>>(N, b);
    LORPC_LAUNCHED();
  } else if (gq) {
    LORPC_TRY(dg_rhs_bc(m, gq, b, s));
  }
  return LORPC_OK;
}

}  // namespace lorpc
