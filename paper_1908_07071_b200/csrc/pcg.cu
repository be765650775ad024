// Preconditioned conjugate gradients (row a10, reading c12).
//
// x_0 = 0, r_0 = b, z = B r, p = z, rho = r.z; per iteration: q = A p,
// alpha = rho / p.q, x += alpha p, r -= alpha q, stop if ||r|| <= rtol ||b||,
// z = B r, rho' = r.z, beta = rho'/rho, p = z + beta p.
// Scalars stay on the device; the dot products are two-stage reductions with a fixed
// grid and tree (deterministic for a given z; the atomics of the operator and patch
// scatters make z itself order-dependent in the last bits).  rho = r.z is fused into
// the last pass over z (the coarse prolongation) when B has its R_0 term; on CG meshes
// the p update also writes the operator's pre-pass (q = p on the Dirichlet nodes, 0
// elsewhere) and in 3D p . q leaves with the element kernel (operator.cu), so an
// iteration has no separate dot-product pass.  On p.Ap <= 0 alpha is set to 0, so a BREAKDOWN return leaves x and r
// as they were.  The host reads ||r|| once per iteration.
#include <cmath>

#include "device.cuh"

namespace lorpc {

enum { S_RHO = 0, S_PQ = 1, S_ALPHA = 2, S_RR = 3, S_RZ = 4, S_BETA = 5, S_BB = 6, S_NS = 8 };
constexpr int RED_BLOCKS = 592;  // 4 x 148 SMs
constexpr int RED_THREADS = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.0;
  if (w == 0) v = warp_sum(v);
  return v;
}

__global__ void k_dot_part(const double* __restrict__ a, const double* __restrict__ b, long long n, double* part) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// mode: 0 rho0, 1 pq (-> alpha), 2 rr, 3 rz (-> beta, rho), 4 bb
__global__ void k_dot_final(const double* __restrict__ part, int np, double* scal, int mode) {
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) {
    switch (mode) {
      case 0: scal[S_RHO] = s; break;
      case 1: scal[S_PQ] = s; scal[S_ALPHA] = s > 0.0 ? scal[S_RHO] / s : 0.0; break;
      case 2: scal[S_RR] = s; break;
      case 3: scal[S_RZ] = s; scal[S_BETA] = s / scal[S_RHO]; scal[S_RHO] = s; break;
      case 4: scal[S_BB] = s; break;
    }
  }
}

// x += alpha p ; r -= alpha q ; partial ||r||^2
__global__ void k_update_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                            const double* __restrict__ q, long long n, const double* __restrict__ scal, double* part) {
  const double alpha = scal[S_ALPHA];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    s += ri * ri;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// CG meshes: p = z + beta p (first: p = z) fused with the operator's pre-pass on its output,
// q = p at the Dirichlet nodes and 0 elsewhere (the element kernel then scatter-adds into q)
template <int DIM>
__global__ void k_update_pq(double* __restrict__ p, const double* __restrict__ z, double* __restrict__ q, int3 N,
                            const double* __restrict__ scal, int first) {
  const double beta = first ? 0.0 : scal[S_BETA];
  const unsigned ndof = (unsigned)N.x * N.y * N.z;
  for (unsigned g = blockIdx.x * blockDim.x + threadIdx.x; g < ndof; g += gridDim.x * blockDim.x) {
    const unsigned gxy = g / (unsigned)N.x;
    const int gx = (int)(g - gxy * N.x), gy = (int)(gxy % (unsigned)N.y), gz = (int)(gxy / (unsigned)N.y);
    bool d = gx == 0 || gx == N.x - 1 || gy == 0 || gy == N.y - 1;
    if (DIM == 3) d = d || gz == 0 || gz == N.z - 1;
    const double pv = first ? z[g] : z[g] + beta * p[g];
    p[g] = pv;
    q[g] = d ? pv : 0.0;
  }
}

// p = z + beta p
__global__ void k_update_p(double* __restrict__ p, const double* __restrict__ z, long long n, const double* __restrict__ scal) {
  const double beta = scal[S_BETA];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

static int dot(const double* a, const double* b, long long n, double* part, double* scal, int mode, cudaStream_t s) {
  k_dot_part<<<RED_BLOCKS, RED_THREADS, 0, s>>>(a, b, n, part);
  LORPC_LAUNCHED();
  k_dot_final<<<1, 1024, 0, s>>>(part, RED_BLOCKS, scal, mode);
  LORPC_LAUNCHED();
  return LORPC_OK;
}

int apply_operator(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s) {
  return m->desc.disc == 0 ? cg_apply(m, x, y, s) : dg_apply(m, x, y, s);
}
int apply_precond(const lorpc_prec* b, const double* r, double* z, cudaStream_t s, double* rzpart);

// z = B r and rho = r.z (mode 0: rho_0; mode 3: beta, rho)
static int precond_rho(const lorpc_prec* b, const double* r, double* z, long long n, double* part, double* scal,
                       int mode, cudaStream_t s) {
  const long long np = rz_parts(b);
  if (np > 0) {
    LORPC_TRY(apply_precond(b, r, z, s, part));
    k_dot_final<<<1, 1024, 0, s>>>(part, (int)np, scal, mode);
    LORPC_LAUNCHED();
    return LORPC_OK;
  }
  LORPC_TRY(apply_precond(b, r, z, s, nullptr));
  return dot(r, z, n, part, scal, mode, s);
}

int pcg_run(const lorpc_mesh* m, const lorpc_prec* b, const double* bvec, double* x, double rtol, int maxit,
            lorpc_pcg_report* rep, cudaStream_t s) {
  const long long n = m->ndof;
  double* r = b->r;
  double* z = b->z;
  double* p = b->pv;
  double* q = b->qv;
  double* scal = b->scal;
  double* part = b->part;
  double* hp = b->hostpin;
  rep->iters = 0; rep->converged = 0; rep->rel_res = 1.0; rep->t_solve_ms = 0.0;
  LORPC_CUDA(cudaEventRecord(b->ev0, s));
  LORPC_CUDA(cudaMemcpyAsync(r, bvec, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  LORPC_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  LORPC_TRY(dot(bvec, bvec, n, part, scal, 4, s));
  LORPC_CUDA(cudaMemcpyAsync(hp, scal, sizeof(double) * S_NS, cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  const double nb = std::sqrt(hp[S_BB]);
  if (rep->res_hist) rep->res_hist[0] = 1.0;
  if (nb == 0.0) {
    rep->converged = 1; rep->rel_res = 0.0;
    LORPC_CUDA(cudaEventRecord(b->ev1, s));
    return LORPC_OK;
  }
  LORPC_TRY(precond_rho(b, r, z, n, part, scal, 0, s));
  // CG meshes: the p update also prepares q for the element kernel; in 3D p . q leaves
  // with the operator (one partial per CTA; p is zero at the Dirichlet nodes in PCG)
  const bool cgm = m->desc.disc == 0 && m->ndof_cg < (1ll << 31);
  const long long nq = cgm ? cg3_blocks(m) : 0;
  const int3 N3 = make_int3(m->N[0], m->N[1], m->N[2]);
  auto update_p = [&](int first) {
    if (cgm) {
      if (m->d == 2) k_update_pq<2><<<RED_BLOCKS, RED_THREADS, 0, s>>>(p, z, q, N3, scal, first);
      else k_update_pq<3><<<RED_BLOCKS, RED_THREADS, 0, s>>>(p, z, q, N3, scal, first);
    } else if (first) {
      return cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s) == cudaSuccess ? LORPC_OK
                                                                                                    : (int)LORPC_ERR_CUDA;
    } else {
      k_update_p<<<RED_BLOCKS, RED_THREADS, 0, s>>>(p, z, n, scal);
    }
    LORPC_LAUNCHED();
    return (int)LORPC_OK;
  };
  LORPC_TRY(update_p(1));
  int status = LORPC_ERR_NOT_CONVERGED;
  for (int k = 1; k <= maxit; ++k) {
    if (cgm) {
      LORPC_TRY(cg_apply_ex(m, p, q, s, false, nq > 0 ? part : nullptr));
      if (nq > 0) {
        k_dot_final<<<1, 1024, 0, s>>>(part, (int)nq, scal, 1);
        LORPC_LAUNCHED();
      } else {
        LORPC_TRY(dot(p, q, n, part, scal, 1, s));
      }
    } else {
      LORPC_TRY(apply_operator(m, p, q, s));
      LORPC_TRY(dot(p, q, n, part, scal, 1, s));
    }
    k_update_xr<<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, r, p, q, n, scal, part);
    LORPC_LAUNCHED();
    k_dot_final<<<1, 1024, 0, s>>>(part, RED_BLOCKS, scal, 2);
    LORPC_LAUNCHED();
    LORPC_CUDA(cudaMemcpyAsync(hp, scal, sizeof(double) * S_NS, cudaMemcpyDeviceToHost, s));
    LORPC_CUDA(cudaStreamSynchronize(s));
    rep->iters = k;
    if (rep->alpha) rep->alpha[k - 1] = hp[S_ALPHA];
    if (k >= 2 && rep->beta) rep->beta[k - 2] = hp[S_BETA];
    if (!(hp[S_PQ] > 0.0)) {
      status = fail(LORPC_ERR_BREAKDOWN, "pcg: p.Ap <= 0 at iteration " + std::to_string(k));
      break;
    }
    const double rel = std::sqrt(hp[S_RR]) / nb;
    rep->rel_res = rel;
    if (rep->res_hist) rep->res_hist[k] = rel;
    if (rel <= rtol) { rep->converged = 1; status = LORPC_OK; break; }
    LORPC_TRY(precond_rho(b, r, z, n, part, scal, 3, s));
    LORPC_TRY(update_p(0));
  }
  LORPC_CUDA(cudaEventRecord(b->ev1, s));
  LORPC_CUDA(cudaEventSynchronize(b->ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, b->ev0, b->ev1);
  rep->t_solve_ms = ms;
  if (status == LORPC_ERR_NOT_CONVERGED) return fail(status, "pcg: not converged in " + std::to_string(maxit));
  return status;
}

}  // namespace lorpc
