// Single-patch preconditioner B(1) (row f2, Table tab:cart-iters):
// "preconditioning the high-order system K_p with an element-structured multigrid
// V-cycle applied to the low-order refined system K_h ... One application of
// MDF-ordered ILU(0) is used for pre-smoothing and post-smoothing at each level.  The
// coarse solve is performed on the p = 1 discretization on the coarse mesh T_p, using
// one V-cycle of BoomerAMG" — here R_0, the GMG V-cycle of reading c11.
//
// The one patch is the whole domain (patch kind 2): its level-l records (ordering,
// L D L^T, DAG schedule) come from the same k_mdf_ilu setup as the vertex patches
// (patch box = all free nodes of the level grid).  The apply runs on the level node
// grids (Dirichlet entries 0): level-scheduled ILU sweeps in one CTA (rows of a DAG
// level in parallel, __syncthreads between levels), residuals with the global level
// stencils, element-structured transfers (the 1D tables of the LOR hierarchy), and
// R_0 on the vertex grid at the bottom.  Sized for the paper's B(1) experiments (at
// most 65535 nodes per level: u16 record offsets); the sweeps use one SM.
#include <algorithm>
#include <cstring>

#include "patch.cuh"

namespace lorpc {

int gmg_vcycle(const lorpc_prec* b, const double** out, cudaStream_t s);

struct SAxis {
  Transfer1D T;
  int ne, Nf, Nc;
};
__device__ __forceinline__ void s_targets(const SAxis& a, int f, int& c0, int& c1, double& w0, double& w1) {
  const int e = min(f / (a.T.mf - 1), a.ne - 1);
  const int t = f - e * (a.T.mf - 1);
  const int base = e * (a.T.mc - 1);
  c0 = base + a.T.c0[t]; c1 = base + a.T.c1[t]; w0 = a.T.w0[t]; w1 = a.T.w1[t];
}

// ---- ILU sweeps on a level grid (one CTA).  Record node indices are box-local
// (box = the free nodes, grid index = box index shifted by one per axis).
template <int DIM>
__global__ void __launch_bounds__(1024) k_single_smooth(const char* __restrict__ rec, int3 Ng, const double* __restrict__ r,
                                                        double* __restrict__ z) {
  const int4 h = *(const int4*)rec;
  const int n = h.x, depth = h.y, nL = h.z;
  const RecLayout R = rec_layout(n, nL);
  const double* D = (const double*)(rec + R.D);
  const double* Lv = (const double*)(rec + R.L);
  const uint16_t* nb = (const uint16_t*)(rec + R.nb);
  const double* bL = (const double*)(rec + R.bL);
  const uint16_t* bk = (const uint16_t*)(rec + R.bk);
  const uint16_t* frp = (const uint16_t*)(rec + R.frp);
  const uint16_t* brp = (const uint16_t*)(rec + R.brp);
  const uint16_t* lpt = (const uint16_t*)(rec + R.lptr);
  const uint16_t* sch = (const uint16_t*)(rec + R.sched);
  const int ex = Ng.x - 2, ey = Ng.y - 2;
  auto gi = [&](int i) {
    const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
    return (long long)(ix + 1) + (long long)Ng.x * ((iy + 1) + (long long)Ng.y * (DIM == 3 ? iz + 1 : 0));
  };
  // forward: w_i = r_i - sum_j L_ij w_j (rows of a DAG level in parallel)
  for (int v = 0; v < depth; ++v) {
    for (int t = lpt[v] + threadIdx.x; t < lpt[v + 1]; t += blockDim.x) {
      const int i = sch[t];
      double a = r[gi(i)];
      for (int e = frp[t]; e < frp[t + 1]; ++e) a -= Lv[e] * z[gi(nb[e])];
      z[gi(i)] = a;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) z[gi(i)] /= D[i];
  __syncthreads();
  // backward: x_i = v_i - sum_k L_ki x_k over the later neighbours k
  for (int v = depth - 1; v >= 0; --v) {
    for (int t = lpt[v] + threadIdx.x; t < lpt[v + 1]; t += blockDim.x) {
      const int i = sch[t];
      double a = z[gi(i)];
      for (int e = brp[t]; e < brp[t + 1]; ++e) a -= bL[e] * z[gi(bk[e])];
      z[gi(i)] = a;
    }
    __syncthreads();
  }
}

// s = r - A z on the interior of a level grid (0 on the boundary)
template <int DIM>
__global__ void k_single_residual(const double* __restrict__ A, const double* __restrict__ r, const double* __restrict__ z,
                                  double* __restrict__ s, int3 Ng) {
  constexpr int ND = Dirs<DIM>::ND;
  const long long NT = (long long)Ng.x * Ng.y * Ng.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NT) return;
  int c[3];
  if (!interior_of<DIM>(g, Ng, c)) { s[g] = 0.0; return; }
  double acc = r[g];
  for (int d = 0; d < ND; ++d) {
    const long long h = g + dir_dx(d) + (long long)Ng.x * (dir_dy(d) + (long long)Ng.y * (DIM == 3 ? dir_dz(d) : 0));
    acc -= A[g * Dirs<DIM>::NDP + d] * z[h];
  }
  s[g] = acc;
}

// r_c += P^T s (scatter from the fine nodes to their <= 2^d coarse parents)
template <int DIM>
__global__ void k_single_restrict(const double* __restrict__ s, double* __restrict__ rc, SAxis ax, SAxis ay, SAxis az) {
  const SAxis* A3[3] = {&ax, &ay, &az};
  const long long NfT = (long long)ax.Nf * ay.Nf * (DIM == 3 ? az.Nf : 1);
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NfT) return;
  const double v = s[g];
  if (v == 0.0) return;
  const int f[3] = {(int)(g % ax.Nf), (int)((g / ax.Nf) % ay.Nf), (int)(g / ((long long)ax.Nf * ay.Nf))};
  int c0[3] = {0, 0, 0}, c1[3] = {0, 0, 0};
  double w0[3] = {1, 1, 1}, w1[3] = {0, 0, 0};
  for (int k = 0; k < DIM; ++k) s_targets(*A3[k], f[k], c0[k], c1[k], w0[k], w1[k]);
  for (int sel = 0; sel < (1 << DIM); ++sel) {
    double w = v;
    long long idx = 0, str = 1;
    bool ok = true;
    for (int k = 0; k < DIM; ++k) {
      const int b = (sel >> k) & 1;
      if (b && c1[k] == c0[k]) { ok = false; break; }
      w *= b ? w1[k] : w0[k];
      idx += (b ? c1[k] : c0[k]) * str;
      str *= A3[k]->Nc;
    }
    if (ok && w != 0.0) atomicAdd(rc + idx, w);
  }
}

// z_f += P e_c on the interior of the fine grid
template <int DIM>
__global__ void k_single_prolong(const double* __restrict__ ec, double* __restrict__ zf, SAxis ax, SAxis ay, SAxis az) {
  const SAxis* A3[3] = {&ax, &ay, &az};
  const long long NfT = (long long)ax.Nf * ay.Nf * (DIM == 3 ? az.Nf : 1);
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NfT) return;
  const int3 Ng = make_int3(ax.Nf, ay.Nf, DIM == 3 ? az.Nf : 1);
  int c[3];
  if (!interior_of<DIM>(g, Ng, c)) return;
  const int f[3] = {(int)(g % ax.Nf), (int)((g / ax.Nf) % ay.Nf), (int)(g / ((long long)ax.Nf * ay.Nf))};
  int c0[3] = {0, 0, 0}, c1[3] = {0, 0, 0};
  double w0[3] = {1, 1, 1}, w1[3] = {0, 0, 0};
  for (int k = 0; k < DIM; ++k) s_targets(*A3[k], f[k], c0[k], c1[k], w0[k], w1[k]);
  double acc = 0.0;
  for (int sel = 0; sel < (1 << DIM); ++sel) {
    double w = 1.0;
    long long idx = 0, str = 1;
    bool ok = true;
    for (int k = 0; k < DIM; ++k) {
      const int b = (sel >> k) & 1;
      if (b && c1[k] == c0[k]) { ok = false; break; }
      w *= b ? w1[k] : w0[k];
      idx += (b ? c1[k] : c0[k]) * str;
      str *= A3[k]->Nc;
    }
    if (ok && w != 0.0) acc += w * ec[idx];
  }
  zf[g] += acc;
}

template <int DIM>
__global__ void k_single_zero_boundary(double* __restrict__ v, int3 Ng) {
  const long long NT = (long long)Ng.x * Ng.y * Ng.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NT) return;
  int c[3];
  if (!interior_of<DIM>(g, Ng, c)) v[g] = 0.0;
}

__global__ void k_single_add(double* __restrict__ z, const double* __restrict__ w, long long n) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g < n) z[g] += w[g];
}

static SAxis saxis(const lorpc_prec* b, int l, int k) {
  SAxis a{};
  a.T = b->lor->T[l];
  a.ne = b->m->n[k];
  a.Nf = b->lor->Nax[l][k];
  a.Nc = b->lor->Nax[l + 1][k];
  return a;
}

// V-cycle on level l: z_l = B_l r_l (level grid vectors, boundary 0)
template <int DIM>
static int single_vcycle(const lorpc_prec* b, int l, const double* r, double* z, cudaStream_t s) {
  const lorpc_lor* lor = b->lor;
  const int L = b->L;
  const int3 Ng = make_int3(lor->Nax[l][0], lor->Nax[l][1], DIM == 3 ? lor->Nax[l][2] : 1);
  const long long NT = lor->Nl[l];
  if (l == L - 1) {  // bottom: R_0 (GMG level 0 = this vertex grid)
    LORPC_CUDA(cudaMemcpyAsync(b->cr[0], r, sizeof(double) * NT, cudaMemcpyDeviceToDevice, s));
    const double* z0 = nullptr;
    LORPC_TRY(gmg_vcycle(b, &z0, s));
    LORPC_CUDA(cudaMemcpyAsync(z, z0, sizeof(double) * NT, cudaMemcpyDeviceToDevice, s));
    return LORPC_OK;
  }
  const char* rec = b->rec + b->recoff_h[l];
  double* sv = b->sgl[l];
  double* wv = b->sgw[l];
  LORPC_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * NT, s));
  k_single_smooth<DIM><<<1, 1024, 0, s>>>(rec, Ng, r, z);                              // pre-smoothing
  LORPC_LAUNCHED();
  k_single_residual<DIM><<<nb(NT, 256), 256, 0, s>>>(lor->A[l], r, z, sv, Ng);
  LORPC_LAUNCHED();
  const long long NC = lor->Nl[l + 1];
  double* rc = b->sgr[l + 1];
  double* ec = b->sgz[l + 1];
  LORPC_CUDA(cudaMemsetAsync(rc, 0, sizeof(double) * NC, s));
  const SAxis ax = saxis(b, l, 0), ay = saxis(b, l, 1), az = DIM == 3 ? saxis(b, l, 2) : SAxis{};
  k_single_restrict<DIM><<<nb(NT, 256), 256, 0, s>>>(sv, rc, ax, ay, az);
  LORPC_LAUNCHED();
  const int3 Nc = make_int3(lor->Nax[l + 1][0], lor->Nax[l + 1][1], DIM == 3 ? lor->Nax[l + 1][2] : 1);
  k_single_zero_boundary<DIM><<<nb(NC, 256), 256, 0, s>>>(rc, Nc);
  LORPC_LAUNCHED();
  LORPC_TRY(single_vcycle<DIM>(b, l + 1, rc, ec, s));
  k_single_prolong<DIM><<<nb(NT, 256), 256, 0, s>>>(ec, z, ax, ay, az);
  LORPC_LAUNCHED();
  k_single_residual<DIM><<<nb(NT, 256), 256, 0, s>>>(lor->A[l], r, z, sv, Ng);
  LORPC_LAUNCHED();
  LORPC_CUDA(cudaMemsetAsync(wv, 0, sizeof(double) * NT, s));
  k_single_smooth<DIM><<<1, 1024, 0, s>>>(rec, Ng, sv, wv);                            // post-smoothing
  LORPC_LAUNCHED();
  k_single_add<<<nb(NT, 256), 256, 0, s>>>(z, wv, NT);
  LORPC_LAUNCHED();
  return LORPC_OK;
}

// z = B(1) r on the CG node grid (level 0 grid = the mesh's node grid); z_D = 0
int single_apply(const lorpc_prec* b, const double* r, double* z, cudaStream_t s) {
  const lorpc_mesh* m = b->m;
  const long long N0 = b->lor->Nl[0];
  double* r0 = b->sgr[0];
  LORPC_CUDA(cudaMemcpyAsync(r0, r, sizeof(double) * N0, cudaMemcpyDeviceToDevice, s));
  const int3 Ng = make_int3(m->N[0], m->N[1], m->N[2]);
  if (m->d == 2) {
    k_single_zero_boundary<2><<<nb(N0, 256), 256, 0, s>>>(r0, Ng);
    LORPC_LAUNCHED();
    return single_vcycle<2>(b, 0, r0, z, s);
  }
  k_single_zero_boundary<3><<<nb(N0, 256), 256, 0, s>>>(r0, Ng);
  LORPC_LAUNCHED();
  return single_vcycle<3>(b, 0, r0, z, s);
}

int single_setup(lorpc_prec* b) {
  for (int l = 0; l < b->L; ++l) {
    const long long n = b->lor->Nl[l];
    LORPC_TRY(dalloc(&b->sgr[l], (size_t)n));
    LORPC_TRY(dalloc(&b->sgz[l], (size_t)n));
    LORPC_TRY(dalloc(&b->sgl[l], (size_t)n));
    LORPC_TRY(dalloc(&b->sgw[l], (size_t)n));
  }
  return LORPC_OK;
}

}  // namespace lorpc
