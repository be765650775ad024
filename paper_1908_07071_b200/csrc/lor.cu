// Low-order-refined operator and the element-structured hierarchy (row a11).
//
// K_h: Q1 stiffness on every GLL subcell, the subcell map being the
// multilinear interpolation of its corner images (= the element map restricted,
// reading c2), integrated with 2^d Gauss points.  Assembled node-parallel
// (each node sums the rows of its <= 2^d incident subcells, no atomics) into a
// full 3^d stencil [ND][N], entry (d, g) = K_h(g, g + offset(d)).
//
// Hierarchy (readings c3/c4): level l+1 keeps every other interior
// GLL point per element (chain from basis.cpp); P_l interpolates linearly in the
// GLL reference coordinate; A_{l+1} = P_l^T A_l P_l computed coarse-node-parallel
// directly in stencil form.  The same Galerkin kernel builds the 2:1
// vertex-centred GMG levels of R_0 (reading c11).
#include "device.cuh"

namespace lorpc {

template <int DIM>
__global__ void k_assemble_kh(const double* __restrict__ X, int3 N, double* __restrict__ A,
                              const double* __restrict__ bsub) {
  constexpr int ND = Dirs<DIM>::ND, NC = 1 << DIM;
  const long long Ntot = (long long)N.x * N.y * N.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= Ntot) return;
  const int gc[3] = {(int)(g % N.x), (int)((g / N.x) % N.y), (int)(g / ((long long)N.x * N.y))};
  const int Nn[3] = {N.x, N.y, N.z};
  double row[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) row[d] = 0.0;
  const double gp[2] = {0.5 - 0.5 / sqrt(3.0), 0.5 + 0.5 / sqrt(3.0)};
  const double wgt = DIM == 2 ? 0.25 : 0.125;
  for (int cme = 0; cme < NC; ++cme) {           // this node is corner `cme` of subcell s = g - cb
    const int cb[3] = {cme & 1, (cme >> 1) & 1, (cme >> 2) & 1};
    int sc[3];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < DIM; ++k) { sc[k] = gc[k] - cb[k]; if (sc[k] < 0 || sc[k] > Nn[k] - 2) ok = false; }
    if (!ok) continue;
    double Xc[NC][DIM];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int cc[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
      const long long id = (sc[0] + cc[0]) + (long long)N.x * ((sc[1] + cc[1]) + (long long)N.y * (DIM == 3 ? sc[2] + cc[2] : 0));
#pragma unroll
      for (int i = 0; i < DIM; ++i) Xc[c][i] = X[id * DIM + i];
    }
    double Kr[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) Kr[c] = 0.0;
    // b at this subcell's Gauss points (row f3; global subcell index)
    const long long sidx = sc[0] + (long long)(N.x - 1) * (sc[1] + (long long)(N.y - 1) * (DIM == 3 ? sc[2] : 0));
#pragma unroll
    for (int ig = 0; ig < NC; ++ig) {
      const int gb[3] = {ig & 1, (ig >> 1) & 1, (ig >> 2) & 1};
      double t[3];
#pragma unroll
      for (int k = 0; k < DIM; ++k) t[k] = gp[gb[k]];
      double J[DIM * DIM], Ji[DIM * DIM], gr[NC][DIM];
#pragma unroll
      for (int i = 0; i < DIM * DIM; ++i) J[i] = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int cc[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          double v = cc[k] ? 1.0 : -1.0;
#pragma unroll
          for (int mm = 0; mm < DIM; ++mm) if (mm != k) v *= cc[mm] ? t[mm] : 1.0 - t[mm];
          gr[c][k] = v;
#pragma unroll
          for (int i = 0; i < DIM; ++i) J[i * DIM + k] += Xc[c][i] * v;
        }
      }
      const double det = inv_det<DIM>(J, Ji);
      double pm[DIM];  // physical gradient of my corner function
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) v += Ji[k * DIM + i] * gr[cme][k];
        pm[i] = v;
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
          double v = 0.0;
#pragma unroll
          for (int k = 0; k < DIM; ++k) v += Ji[k * DIM + i] * gr[c][k];
          s += pm[i] * v;
        }
        Kr[c] += (bsub ? wgt * bsub[sidx * NC + ig] : wgt) * det * s;
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int cc[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
      int dd = (cc[0] - cb[0] + 1) + 3 * (cc[1] - cb[1] + 1);
      if (DIM == 3) dd += 9 * (cc[2] - cb[2] + 1);
      row[dd] += Kr[c];
    }
  }
#pragma unroll
  for (int d = 0; d < ND; ++d) A[g * Dirs<DIM>::NDP + d] = row[d];
  A[g * Dirs<DIM>::NDP + ND] = 0.0;
}

// weight of coarse 1D index ic in the interpolation row of fine 1D index f
struct Axis1D {
  Transfer1D T;
  int ne;  // elements (coarse intervals) along the axis
  int Nf, Nc;
};
__device__ __forceinline__ void fine_targets(const Axis1D& a, int f, int& c0, int& c1, double& w0, double& w1) {
  const int e = min(f / (a.T.mf - 1), a.ne - 1);
  const int t = f - e * (a.T.mf - 1);
  const int base = e * (a.T.mc - 1);
  c0 = base + a.T.c0[t]; c1 = base + a.T.c1[t]; w0 = a.T.w0[t]; w1 = a.T.w1[t];
}
__device__ __forceinline__ double pweight(const Axis1D& a, int f, int ic) {
  int c0, c1; double w0, w1;
  fine_targets(a, f, c0, c1, w0, w1);
  double w = 0.0;
  if (c0 == ic) w += w0;
  if (c1 == ic && c1 != c0) w += w1;
  return w;
}
__device__ __forceinline__ int fine_pos(const Axis1D& a, int ic) {
  const int e = min(ic / (a.T.mc - 1), a.ne - 1);
  const int t = ic - e * (a.T.mc - 1);
  return e * (a.T.mf - 1) + a.T.ret[t];
}

template <int DIM>
__global__ void k_galerkin(const double* __restrict__ Af, double* __restrict__ Ac, Axis1D ax, Axis1D ay, Axis1D az) {
  constexpr int ND = Dirs<DIM>::ND;
  const Axis1D* A3[3] = {&ax, &ay, &az};
  const long long Ncx = ax.Nc, Ncy = ay.Nc, Ncz = DIM == 3 ? az.Nc : 1;
  const long long Nfx = ax.Nf, Nfy = ay.Nf, Nfz = DIM == 3 ? az.Nf : 1;
  const long long NcT = Ncx * Ncy * Ncz;
  const long long I = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (I >= NcT) return;
  const int Ic[3] = {(int)(I % Ncx), (int)((I / Ncx) % Ncy), (int)(I / (Ncx * Ncy))};
  double row[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) row[d] = 0.0;
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  const int Nf3[3] = {(int)Nfx, (int)Nfy, (int)Nfz};
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    const int fp = fine_pos(*A3[k], Ic[k]);
    lo[k] = max(fp - A3[k]->T.gap, 0);
    hi[k] = min(fp + A3[k]->T.gap, Nf3[k] - 1);
  }
  for (int fz = lo[2]; fz <= hi[2]; ++fz) {
    const double wz = DIM == 3 ? pweight(az, fz, Ic[2]) : 1.0;
    if (wz == 0.0) continue;
    for (int fy = lo[1]; fy <= hi[1]; ++fy) {
      const double wy = pweight(ay, fy, Ic[1]);
      if (wy == 0.0) continue;
      for (int fx = lo[0]; fx <= hi[0]; ++fx) {
        const double wx = pweight(ax, fx, Ic[0]);
        if (wx == 0.0) continue;
        const double wa = wx * wy * wz;
        const long long a = fx + Nfx * (fy + Nfy * fz);
        for (int d = 0; d < ND; ++d) {
          const int b[3] = {fx + dir_dx(d), fy + dir_dy(d), fz + (DIM == 3 ? dir_dz(d) : 0)};
          if (b[0] < 0 || b[0] >= Nfx || b[1] < 0 || b[1] >= Nfy) continue;
          if (DIM == 3 && (b[2] < 0 || b[2] >= Nfz)) continue;
          const double av = Af[a * Dirs<DIM>::NDP + d];
          if (av == 0.0) continue;
          int c0[3], c1[3]; double w0[3], w1[3];
#pragma unroll
          for (int k = 0; k < DIM; ++k) fine_targets(*A3[k], b[k], c0[k], c1[k], w0[k], w1[k]);
          // enumerate the <= 2^d coarse targets of b
          for (int sel = 0; sel < (1 << DIM); ++sel) {
            double w = wa * av;
            int off[3] = {0, 0, 0};
            bool ok = true;
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
              const int s = (sel >> k) & 1;
              const int c = s ? c1[k] : c0[k];
              const double ww = s ? w1[k] : w0[k];
              if (s && c1[k] == c0[k]) { ok = false; break; }
              if (ww == 0.0) { ok = false; break; }
              w *= ww;
              off[k] = c - Ic[k];
              if (off[k] < -1 || off[k] > 1) { ok = false; break; }
            }
            if (!ok) continue;
            int dd = (off[0] + 1) + 3 * (off[1] + 1);
            if (DIM == 3) dd += 9 * (off[2] + 1);
            row[dd] += w;
          }
        }
      }
    }
  }
#pragma unroll
  for (int d = 0; d < ND; ++d) Ac[I * Dirs<DIM>::NDP + d] = row[d];
  Ac[I * Dirs<DIM>::NDP + ND] = 0.0;
}

static Transfer1D make_transfer(const double* xi, const std::vector<int>& fine, const std::vector<int>& coarse) {
  Transfer1D T{};
  T.mf = (int)fine.size(); T.mc = (int)coarse.size();
  int maxgap = 0;
  for (int t = 0; t < T.mf; ++t) {
    const int a = fine[t];
    int hit = -1;
    for (int c = 0; c < T.mc; ++c) if (coarse[c] == a) hit = c;
    if (hit >= 0) { T.c0[t] = T.c1[t] = hit; T.w0[t] = 1.0; T.w1[t] = 0.0; continue; }
    int c = 0;
    while (!(coarse[c] < a && a < coarse[c + 1])) ++c;
    const double xl = xi[coarse[c]], xh = xi[coarse[c + 1]], xa = xi[a];
    T.c0[t] = c; T.c1[t] = c + 1;
    T.w0[t] = (xh - xa) / (xh - xl); T.w1[t] = (xa - xl) / (xh - xl);
  }
  for (int c = 0; c < T.mc; ++c) {
    for (int t = 0; t < T.mf; ++t) if (fine[t] == coarse[c]) T.ret[c] = t;
    if (c > 0) maxgap = std::max(maxgap, T.ret[c] - T.ret[c - 1]);
  }
  T.gap = maxgap;
  return T;
}

Transfer1D gmg_transfer() {
  Transfer1D T{};
  T.mf = 3; T.mc = 2; T.gap = 2;
  T.c0[0] = T.c1[0] = 0; T.w0[0] = 1.0; T.w1[0] = 0.0;
  T.c0[1] = 0; T.c1[1] = 1; T.w0[1] = 0.5; T.w1[1] = 0.5;
  T.c0[2] = T.c1[2] = 1; T.w0[2] = 1.0; T.w1[2] = 0.0;
  T.ret[0] = 0; T.ret[1] = 2;
  return T;
}

int galerkin(int d, const double* Af, double* Ac, const Transfer1D& T, const int* ne, const int* Nf, const int* Nc,
             cudaStream_t s) {
  Axis1D a[3];
  long long NcT = 1;
  for (int k = 0; k < 3; ++k) {
    a[k].T = T; a[k].ne = ne[k]; a[k].Nf = Nf[k]; a[k].Nc = Nc[k];
    if (k < d) NcT *= Nc[k];
  }
  const unsigned g = (unsigned)((NcT + 127) / 128);
  if (d == 2) k_galerkin<2><<<g, 128, 0, s>>>(Af, Ac, a[0], a[1], a[2]);
  else k_galerkin<3><<<g, 128, 0, s>>>(Af, Ac, a[0], a[1], a[2]);
  LORPC_LAUNCHED();
  return LORPC_OK;
}

int lor_build(const lorpc_mesh* m, lorpc_lor* l, cudaStream_t s) {
  const int d = m->d;
  auto ch = make_chain(m->p);
  l->m = m;
  l->L = (int)ch.size();
  if (l->L > MAXL) return fail(LORPC_ERR_SIZE, "too many levels");
  for (int i = 0; i < MAXL; ++i) l->A[i] = nullptr;
  for (int lv = 0; lv < l->L; ++lv) {
    l->ml[lv] = (int)ch[lv].size();
    l->Nl[lv] = 1;
    for (int k = 0; k < 3; ++k) {
      l->Nax[lv][k] = (k < d) ? m->n[k] * (l->ml[lv] - 1) + 1 : 1;
      l->Nl[lv] *= l->Nax[lv][k];
    }
    LORPC_TRY(dalloc(&l->A[lv], (size_t)ndp_of(d) * l->Nl[lv]));
    if (lv + 1 < l->L) l->T[lv] = make_transfer(m->basis.xi, ch[lv], ch[lv + 1]);
  }
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  const unsigned g = (unsigned)((m->ndof_cg + 127) / 128);
  if (d == 2) k_assemble_kh<2><<<g, 128, 0, s>>>(m->X, N, l->A[0], m->bsub);
  else k_assemble_kh<3><<<g, 128, 0, s>>>(m->X, N, l->A[0], m->bsub);
  LORPC_LAUNCHED();
  for (int lv = 0; lv + 1 < l->L; ++lv)
    LORPC_TRY(galerkin(d, l->A[lv], l->A[lv + 1], l->T[lv], m->n, l->Nax[lv], l->Nax[lv + 1], s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  return LORPC_OK;
}

}  // namespace lorpc
