// C ABI (include/lorpc.h): argument checking, handle lifetime, dispatch.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "device.cuh"

namespace lorpc {
const char* last_error();
int apply_operator(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s);
int export_ordering(const lorpc_prec* b, long long j, int l, int* perm, int* n);

int apply_precond(const lorpc_prec* b, const double* r, double* z, cudaStream_t s, double* rzpart) {
  if (b->m->desc.disc == 0) return schwarz_apply_cg(b, r, z, s, rzpart);
  LORPC_TRY(dg_restrict_cg(b->m, r, b->rcg, s));
  LORPC_TRY(schwarz_apply_cg(b, b->rcg, b->zcg, s));
  return dg_combine(b->m, r, b->zcg, z, s);
}
// r.z can ride on the last pass over z (the coarse prolongation) for CG with R_0
long long rz_parts(const lorpc_prec* b) {
  return (b->m->desc.disc == 0 && b->desc.coarse == 0 && b->desc.patch_kind != 2) ? (b->m->ndof_cg + 255) / 256 : 0;
}
}  // namespace lorpc

using namespace lorpc;

static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

extern "C" {

const char* lorpc_last_error(void) { return lorpc::last_error(); }

long long lorpc_launch_count(int reset) {
  long long v = launch_counter();
  if (reset) launch_counter() = 0;
  return v;
}

int lorpc_mesh_create(const lorpc_mesh_desc* desc, const double* vertices_host, void* stream, lorpc_mesh** out) {
  if (!desc || !vertices_host || !out) return fail(LORPC_ERR_ARG, "mesh_create: NULL argument");
  *out = nullptr;
  const int d = desc->dim;
  if (d != 2 && d != 3) return fail(LORPC_ERR_ARG, "mesh_create: dim must be 2 or 3");
  if (desc->p < 1) return fail(LORPC_ERR_ARG, "mesh_create: p must be >= 1");
  if ((d == 2 && desc->p > 8) || (d == 3 && desc->p > 6)) return fail(LORPC_ERR_SIZE, "mesh_create: p not compiled");
  for (int k = 0; k < d; ++k) if (desc->n[k] < 1) return fail(LORPC_ERR_ARG, "mesh_create: n must be >= 1");
  if (desc->disc < 0 || desc->disc > 2) return fail(LORPC_ERR_ARG, "mesh_create: disc must be 0 (CG), 1 (SIPG), 2 (BR2)");
  if (desc->disc != 0 && !(desc->eta > 0.0)) return fail(LORPC_ERR_ARG, "mesh_create: eta must be > 0");
  if (desc->quad != 0 && desc->quad != 1) return fail(LORPC_ERR_ARG, "mesh_create: quad must be 0 (Gauss) or 1 (GLL)");
  if (desc->quad == 1 && desc->disc != 0) return fail(LORPC_ERR_ARG, "mesh_create: GLL collocation is CG only");
  if (desc->disc != 0 && d != 3) return fail(LORPC_ERR_SIZE, "mesh_create: DG is built for 3D meshes");
  if (desc->disc == 2) {
    // the BR2 lifting kernels use M_K = det J (M1 x M1 x M1): elements must be affine
    // (parallelepipeds): the mixed terms of every trilinear map must vanish
    const int nx = desc->n[0], ny = desc->n[1], nz = desc->n[2];
    auto V = [&](int i, int j, int k, int c) {
      return vertices_host[(((long long)k * (ny + 1) + j) * (nx + 1) + i) * 3 + c];
    };
    for (int k = 0; k < nz; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
          for (int c = 0; c < 3; ++c) {
            const double ex = V(i + 1, j, k, c) - V(i, j, k, c);
            const double sc = std::fabs(ex) + std::fabs(V(i, j + 1, k, c) - V(i, j, k, c)) +
                              std::fabs(V(i, j, k + 1, c) - V(i, j, k, c)) + 1e-300;
            const double mxy = V(i + 1, j + 1, k, c) - V(i + 1, j, k, c) - V(i, j + 1, k, c) + V(i, j, k, c);
            const double mxz = V(i + 1, j, k + 1, c) - V(i + 1, j, k, c) - V(i, j, k + 1, c) + V(i, j, k, c);
            const double myz = V(i, j + 1, k + 1, c) - V(i, j + 1, k, c) - V(i, j, k + 1, c) + V(i, j, k, c);
            if (std::fabs(mxy) + std::fabs(mxz) + std::fabs(myz) > 1e-12 * sc)
              return fail(LORPC_ERR_SIZE, "mesh_create: BR2 needs affine (parallelepiped) elements; element " +
                                              std::to_string(i + (long long)nx * (j + (long long)ny * k)) + " is not");
          }
  }
  lorpc_mesh* m = new lorpc_mesh();
  m->desc = *desc;
  m->d = d; m->p = desc->p; m->q = desc->p + 1;
  m->nloc = 1; m->nq = 1;
  m->nel = 1; m->ndof_cg = 1;
  long long nvert = 1;
  for (int k = 0; k < 3; ++k) {
    m->n[k] = k < d ? desc->n[k] : 1;
    m->N[k] = k < d ? desc->n[k] * desc->p + 1 : 1;
    m->nel *= m->n[k];
    m->ndof_cg *= m->N[k];
    if (k < d) { m->nloc *= m->p + 1; m->nq *= m->q; nvert *= m->n[k] + 1; }
  }
  m->ndof = desc->disc == 0 ? m->ndof_cg : m->nel * m->nloc;
  m->ez_lo = 0; m->ez_hi = m->n[2];
  m->nquad = m->nel * m->nq;
  m->nbq = 0;
  if (desc->disc != 0) {
    long long faces = 0;
    for (int k = 0; k < d; ++k) faces += 2 * (m->nel / m->n[k]);
    m->nbq = faces * (d == 2 ? m->q : m->q * m->q);
  }
  make_basis(m->p, m->basis, desc->quad);
  cudaStream_t s = S(stream);
  int rc = dalloc(&m->V, (size_t)nvert * d);
  if (rc == LORPC_OK) {
    cudaError_t e = cudaMemcpyAsync(m->V, vertices_host, sizeof(double) * nvert * d, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) rc = fail(LORPC_ERR_CUDA, cudaGetErrorString(e));
  }
  if (rc == LORPC_OK) rc = geom_setup(m, s);
  if (rc == LORPC_OK && desc->disc != 0) rc = dg_diag_setup(m, s);
  if (rc != LORPC_OK) { lorpc_mesh_destroy(m); return rc; }
  *out = m;
  return LORPC_OK;
}

void lorpc_mesh_destroy(lorpc_mesh* m) {
  if (!m) return;
  dfree(m->V); dfree(m->G); dfree(m->X); dfree(m->vol); dfree(m->dgdiag); dfree(m->ywork);
  dfree(m->bq); dfree(m->bsub);
  delete m;
}

int lorpc_mesh_sizes(const lorpc_mesh* m, long long* n_dof, long long* n_quad, long long* n_bface_quad) {
  if (!m) return fail(LORPC_ERR_ARG, "mesh_sizes: NULL mesh");
  if (n_dof) *n_dof = m->ndof;
  if (n_quad) *n_quad = m->nquad;
  if (n_bface_quad) *n_bface_quad = m->nbq;
  return LORPC_OK;
}

int lorpc_quad_points(const lorpc_mesh* m, double* xq_dev, double* xbq_dev, void* stream) {
  if (!m) return fail(LORPC_ERR_ARG, "quad_points: NULL mesh");
  if (xbq_dev && m->desc.disc == 0) return fail(LORPC_ERR_ARG, "quad_points: boundary points only for DG");
  return quad_points(m, xq_dev, xbq_dev, S(stream));
}

int lorpc_mesh_set_coefficient(lorpc_mesh* m, const double* bq_dev, const double* bsub_dev, void* stream) {
  if (!m) return fail(LORPC_ERR_ARG, "mesh_set_coefficient: NULL mesh");
  if (m->desc.disc != 0) return fail(LORPC_ERR_ARG, "mesh_set_coefficient: CG meshes only");
  return set_coefficient(m, bq_dev, bsub_dev, S(stream));
}

int lorpc_subcell_points(const lorpc_mesh* m, double* xs_dev, long long* n_sub, void* stream) {
  if (!m) return fail(LORPC_ERR_ARG, "subcell_points: NULL mesh");
  if (n_sub) *n_sub = n_subcells(m);
  if (!xs_dev) return LORPC_OK;
  return subcell_points(m, xs_dev, S(stream));
}

int lorpc_rhs_assemble(const lorpc_mesh* m, const double* fq_dev, const double* gq_dev, double* b_dev, void* stream) {
  if (!m || !fq_dev || !b_dev) return fail(LORPC_ERR_ARG, "rhs_assemble: NULL argument");
  return rhs_assemble(m, fq_dev, gq_dev, b_dev, S(stream));
}

int lorpc_operator_apply(const lorpc_mesh* m, const double* x_dev, double* y_dev, void* stream) {
  if (!m || !x_dev || !y_dev) return fail(LORPC_ERR_ARG, "operator_apply: NULL argument");
  if (x_dev == y_dev) return fail(LORPC_ERR_ARG, "operator_apply: x and y alias");
  return apply_operator(m, x_dev, y_dev, S(stream));
}

int lorpc_lor_assemble(const lorpc_mesh* m, void* stream, lorpc_lor** out) {
  if (!m || !out) return fail(LORPC_ERR_ARG, "lor_assemble: NULL argument");
  *out = nullptr;
  lorpc_lor* l = new lorpc_lor();
  int rc = lor_build(m, l, S(stream));
  if (rc != LORPC_OK) { lorpc_lor_destroy(l); return rc; }
  *out = l;
  return LORPC_OK;
}

void lorpc_lor_destroy(lorpc_lor* l) {
  if (!l) return;
  for (int i = 0; i < MAXL; ++i) dfree(l->A[i]);
  delete l;
}

int lorpc_schwarz_setup(const lorpc_lor* l, const lorpc_schwarz_desc* desc, void* stream, lorpc_prec** out) {
  if (!l || !desc || !out) return fail(LORPC_ERR_ARG, "schwarz_setup: NULL argument");
  if (desc->patch_kind < 0 || desc->patch_kind > 2) return fail(LORPC_ERR_ARG, "schwarz_setup: patch_kind");
  if (desc->ordering < 0 || desc->ordering > 2) return fail(LORPC_ERR_ARG, "schwarz_setup: ordering");
  if (desc->coarse < 0 || desc->coarse > 1) return fail(LORPC_ERR_ARG, "schwarz_setup: coarse");
  if (desc->extend < 0 || desc->extend > 1) return fail(LORPC_ERR_ARG, "schwarz_setup: extend");
  *out = nullptr;
  lorpc_prec* b = new lorpc_prec();
  b->lor = l; b->m = l->m; b->desc = *desc;
  for (int i = 0; i < MAXC; ++i) { b->Ac[i] = b->dl1[i] = b->cr[i] = b->cz[i] = b->cs[i] = nullptr; }
  cudaStream_t s = S(stream);
  int rc = schwarz_build(b, s);
  const lorpc_mesh* m = b->m;
  if (rc == LORPC_OK && m->desc.disc != 0) {
    rc = dalloc(&b->rcg, (size_t)m->ndof_cg);
    if (rc == LORPC_OK) rc = dalloc(&b->zcg, (size_t)m->ndof_cg);
  }
  if (rc == LORPC_OK) rc = dalloc(&b->r, (size_t)m->ndof);
  if (rc == LORPC_OK) rc = dalloc(&b->z, (size_t)m->ndof);
  if (rc == LORPC_OK) rc = dalloc(&b->pv, (size_t)m->ndof);
  if (rc == LORPC_OK) rc = dalloc(&b->qv, (size_t)m->ndof);
  if (rc == LORPC_OK) rc = dalloc(&b->scal, 16);
  b->npart = std::max<long long>(std::max<long long>(1024, rz_parts(b)), cg3_blocks(m));
  if (rc == LORPC_OK) rc = dalloc(&b->part, (size_t)b->npart);
  if (rc == LORPC_OK && cudaMallocHost(&b->hostpin, 16 * sizeof(double)) != cudaSuccess)
    rc = fail(LORPC_ERR_OOM, "cudaMallocHost");
  if (rc == LORPC_OK && (cudaEventCreate(&b->ev0) != cudaSuccess || cudaEventCreate(&b->ev1) != cudaSuccess ||
                         cudaEventCreateWithFlags(&b->evf, cudaEventDisableTiming) != cudaSuccess ||
                         cudaEventCreateWithFlags(&b->evj, cudaEventDisableTiming) != cudaSuccess))
    rc = fail(LORPC_ERR_CUDA, "cudaEventCreate");
  if (rc == LORPC_OK && cudaStreamCreateWithFlags(&b->aux, cudaStreamNonBlocking) != cudaSuccess)
    rc = fail(LORPC_ERR_CUDA, "cudaStreamCreate");
  if (rc != LORPC_OK) { lorpc_prec_destroy(b); return rc; }
  *out = b;
  return LORPC_OK;
}

void lorpc_prec_destroy(lorpc_prec* b) {
  if (!b) return;
  dfree(b->rec); dfree(b->recoff); dfree(b->trec); dfree(b->trecoff); dfree(b->zpark); dfree(b->Cdi); dfree(b->pord);
  dfree(b->wrec); dfree(b->wrecoff); dfree(b->Cq); dfree(b->erng);
  dfree(b->qrec); dfree(b->qrecoff); dfree(b->qsched);
  for (int l = 0; l < MAXL; ++l) { dfree(b->sgr[l]); dfree(b->sgz[l]); dfree(b->sgl[l]); dfree(b->sgw[l]); }
  for (int i = 0; i < MAXC; ++i) {
    if (i > 0) dfree(b->Ac[i]);
    dfree(b->dl1[i]); dfree(b->cr[i]); dfree(b->cz[i]); dfree(b->cs[i]);
  }
  dfree(b->coarse_chol); dfree(b->coarse_idx); dfree(b->rcg); dfree(b->zcg); dfree(b->xb); dfree(b->wtab); dfree(b->Cd);
  dfree(b->r); dfree(b->z); dfree(b->pv); dfree(b->qv); dfree(b->scal); dfree(b->part);
  if (b->hostpin) cudaFreeHost(b->hostpin);
  if (b->ev0) cudaEventDestroy(b->ev0);
  if (b->ev1) cudaEventDestroy(b->ev1);
  if (b->evf) cudaEventDestroy(b->evf);
  if (b->evj) cudaEventDestroy(b->evj);
  if (b->aux) cudaStreamDestroy(b->aux);
  for (auto& e : b->prof_ev) cudaEventDestroy(e);
  delete b;
}

int lorpc_precond_apply(const lorpc_prec* b, const double* r_dev, double* z_dev, void* stream) {
  if (!b || !r_dev || !z_dev) return fail(LORPC_ERR_ARG, "precond_apply: NULL argument");
  if (r_dev == z_dev) return fail(LORPC_ERR_ARG, "precond_apply: r and z alias");
  return apply_precond(b, r_dev, z_dev, S(stream), nullptr);
}

int lorpc_prec_export_ordering(const lorpc_prec* b, long long patch, int level, int* perm_host, int* n) {
  if (!b || !perm_host || !n) return fail(LORPC_ERR_ARG, "export_ordering: NULL argument");
  return export_ordering(b, patch, level, perm_host, n);
}

int lorpc_prec_info(const lorpc_prec* b, long long* n_patches, int* n_levels) {
  if (!b) return fail(LORPC_ERR_ARG, "prec_info: NULL");
  if (n_patches) *n_patches = b->J;
  if (n_levels) *n_levels = b->L;
  return LORPC_OK;
}

int lorpc_prec_kernel(const lorpc_prec* b, int* mode) {
  if (!b || !mode) return fail(LORPC_ERR_ARG, "prec_kernel: NULL");
  *mode = b->qmode ? 4 : b->wmode ? 2 : b->umode ? 3 : b->tmode ? 1 : 0;
  return LORPC_OK;
}

int lorpc_prec_bytes(const lorpc_prec* b, long long* factor_values, long long* level_nodes, long long* coarse_nodes) {
  if (!b) return fail(LORPC_ERR_ARG, "prec_bytes: NULL");
  if (factor_values) *factor_values = b->factor_values;
  if (level_nodes)
    for (int l = 0; l < b->L; ++l) level_nodes[l] = b->lor->Nl[l];
  if (coarse_nodes) {
    long long c = 0;
    for (int l = 0; l < b->nc; ++l) c += b->cN[l];
    *coarse_nodes = c;
  }
  return LORPC_OK;
}

int lorpc_prec_profile(lorpc_prec* b, int enable) {
  if (!b) return fail(LORPC_ERR_ARG, "prec_profile: NULL");
  if (enable && b->prof_ev.empty()) {
    b->prof_ev.resize(8192);
    for (auto& e : b->prof_ev) LORPC_CUDA(cudaEventCreate(&e));
  }
  b->prof_on = enable != 0;
  return LORPC_OK;
}

int lorpc_prec_profile_read(lorpc_prec* b, double* ms, long long* launches) {
  if (!b || !ms || !launches) return fail(LORPC_ERR_ARG, "prec_profile_read: NULL");
  double acc = 0.0;
  for (int i = 0; i < b->prof_n; ++i) {
    LORPC_CUDA(cudaEventSynchronize(b->prof_ev[2 * i + 1]));
    float t = 0.f;
    LORPC_CUDA(cudaEventElapsedTime(&t, b->prof_ev[2 * i], b->prof_ev[2 * i + 1]));
    acc += t;
  }
  *ms = acc;
  *launches = b->prof_n;
  b->prof_n = 0;
  return LORPC_OK;
}

int lorpc_pcg_solve(const lorpc_mesh* m, const lorpc_prec* b, const double* b_dev, double* x_dev, double rtol,
                    int maxit, lorpc_pcg_report* rep, void* stream) {
  if (!m || !b || !b_dev || !x_dev || !rep) return fail(LORPC_ERR_ARG, "pcg_solve: NULL argument");
  if (b->m != m) return fail(LORPC_ERR_ARG, "pcg_solve: preconditioner built for another mesh");
  if (!(rtol > 0.0) || maxit < 1) return fail(LORPC_ERR_ARG, "pcg_solve: rtol > 0 and maxit >= 1 required");
  return pcg_run(m, b, b_dev, x_dev, rtol, maxit, rep, S(stream));
}

int lorpc_pcg_solve_host(const lorpc_mesh* m, const lorpc_prec* b, const double* b_host, double* x_host, double rtol,
                         int maxit, lorpc_pcg_report* rep, void* stream) {
  if (!m || !b || !b_host || !x_host || !rep) return fail(LORPC_ERR_ARG, "pcg_solve_host: NULL argument");
  if (b->m != m) return fail(LORPC_ERR_ARG, "pcg_solve_host: preconditioner built for another mesh");
  if (!(rtol > 0.0) || maxit < 1) return fail(LORPC_ERR_ARG, "pcg_solve_host: rtol > 0 and maxit >= 1 required");
  cudaStream_t s = S(stream);
  lorpc_prec* bb = const_cast<lorpc_prec*>(b);
  if (bb->xb && bb->xb_n != m->ndof) { dfree(bb->xb); bb->xb_n = 0; }
  if (!bb->xb) { LORPC_TRY(dalloc(&bb->xb, (size_t)2 * m->ndof)); bb->xb_n = m->ndof; }
  double* bd = bb->xb;
  double* xd = bb->xb + m->ndof;
  LORPC_CUDA(cudaMemcpyAsync(bd, b_host, sizeof(double) * m->ndof, cudaMemcpyHostToDevice, s));
  int rc = pcg_run(m, b, bd, xd, rtol, maxit, rep, s);
  if (rc != LORPC_OK && rc != LORPC_ERR_NOT_CONVERGED) return rc;
  LORPC_CUDA(cudaMemcpyAsync(x_host, xd, sizeof(double) * m->ndof, cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  return rc;
}

}  // extern "C"
