// Multi-GPU slab decomposition of the CG path (BASELINE C5:
// "element slabs partitioned across 1/2/4/8 GPUs with NCCL halo exchange").
//
// Rank r owns element layers [z0, z1) along z (the slowest axis), node planes
// [z0 p, z1 p) and vertex planes [z0, z1) (the last rank also the top plane).  It
// holds a local sub-mesh of element layers [za, zb) = [z0 - 1, z1 + 1] clipped to
// the domain: one ghost element layer on each side, built from the replicated
// vertex array, so that every LOR row, patch factor and coarse row a rank needs
// is computed locally (no communication in setup except the coarse gather).
//
// One PCG iteration exchanges, over NCCL point-to-point between slab
// neighbours:
//   E1  operator input   p on plane z1 p          (rank r+1 -> r, copy)
//   E2  operator output  partial A p on z1 p       (rank r -> r+1, add)
//   E3  Schwarz input    r on planes z0 p - p+1 .. z0 p - 1   (rank r-1 -> r, copy)
//   E4  Schwarz output   patch sums on those planes (rank r -> r-1, add)
// plus one allreduce of the coarse residual on the global vertex grid (each rank
// restricts its owned vertex planes, eq:as j = 0 term; R_0 then runs replicated on
// every rank, reading c11) and the scalar allreduces of the dot products.
//
// The same code runs R ranks inside one process on one device ("emulation": the
// exchanges become device copies and the reductions a fixed-order sum over the
// ranks' partials), which is how the multi-rank path is tested without R GPUs.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "patch.cuh"

struct lorpc_dist;

namespace lorpc {

constexpr int DRED_BLOCKS = 296, DRED_THREADS = 256;
enum { D_BB = 0, D_RHO = 1, D_PQ = 2, D_RR = 3, D_RZ = 4, D_NS = 8 };

__device__ __forceinline__ double dblock_sum(double v) {
  __shared__ double sh[32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.0;
  if (w == 0) v = warp_sum(v);
  return v;
}
__global__ void k_ddot(const double* __restrict__ a, const double* __restrict__ b, long long n, double* part) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  s = dblock_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_dsum(const double* __restrict__ part, int np, double* out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = dblock_sum(s);
  if (threadIdx.x == 0) *out = s;
}
// emulation allreduce: fixed-order sum of slot k over the ranks' local scalars
__global__ void k_rank_sum(double* const* loc, double* const* glob, int R, int k) {
  double s = 0.0;
  for (int r = 0; r < R; ++r) s += loc[r][k];
  for (int r = 0; r < R; ++r) glob[r][k] = s;
}
// x += alpha p, r -= alpha q with alpha = rho / pq (global scalars)
__global__ void k_dupdate_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ q, long long n, const double* __restrict__ S) {
  const double alpha = S[D_RHO] / S[D_PQ];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    r[i] -= alpha * q[i];
  }
}
// p = z + beta p with beta = rz / rho; then rho = rz
__global__ void k_dupdate_p(double* __restrict__ p, const double* __restrict__ z, long long n, const double* S) {
  const double beta = S[D_RZ] / S[D_RHO];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}
__global__ void k_dset(double* S, int dst, int src) { S[dst] = S[src]; }
// dst += src on nplanes planes of Nx x Ny nodes, skipping the (Dirichlet) side faces
__global__ void k_add_planes_free(double* __restrict__ dst, const double* __restrict__ src, int Nx, int Ny, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int gx = (int)(i % Nx), gy = (int)((i / Nx) % Ny);
  if (gx == 0 || gx == Nx - 1 || gy == 0 || gy == Ny - 1) return;
  dst[i] += src[i];
}
// coarse residual r_c = P_0^T r at the vertices of local vertex planes [v0, v1)
// (the restriction of k_restrict_vertex; boundary vertices of the GLOBAL grid hold 0)
__global__ void k_restrict_vertex_planes(const double* __restrict__ r, double* __restrict__ rc, int3 nv, int3 N,
                                         Basis1D bs, int v0, int v1, int gz0, int gnvz) {
  const long long per = (long long)nv.x * nv.y;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= per * (v1 - v0)) return;
  const long long v = t + per * v0;
  const int vc[3] = {(int)(v % nv.x), (int)((v / nv.x) % nv.y), (int)(v / per)};
  const int gzv = vc[2] + gz0;
  if (vc[0] == 0 || vc[0] == nv.x - 1 || vc[1] == 0 || vc[1] == nv.y - 1 || gzv == 0 || gzv == gnvz - 1) {
    rc[v] = 0.0;
    return;
  }
  const int p = bs.p;
  double acc = 0.0;
  for (int gz = (vc[2] - 1) * p + 1; gz <= (vc[2] + 1) * p - 1; ++gz) {
    const int tz = gz - vc[2] * p;
    const double wz = tz <= 0 ? bs.xi[tz + p] : 1.0 - bs.xi[tz];
    for (int gy = (vc[1] - 1) * p + 1; gy <= (vc[1] + 1) * p - 1; ++gy) {
      const int ty = gy - vc[1] * p;
      const double wy = ty <= 0 ? bs.xi[ty + p] : 1.0 - bs.xi[ty];
      for (int gx = (vc[0] - 1) * p + 1; gx <= (vc[0] + 1) * p - 1; ++gx) {
        const int tx = gx - vc[0] * p;
        const double wx = tx <= 0 ? bs.xi[tx + p] : 1.0 - bs.xi[tx];
        acc += wx * wy * wz * r[gx + (long long)N.x * (gy + (long long)N.y * gz)];
      }
    }
  }
  rc[v] = acc;
}

}  // namespace lorpc

using namespace lorpc;

struct DistRank {
  int rank = 0;
  lorpc_dist_plan plan{};
  int z0 = 0, z1 = 0, za = 0, zb = 0;  // owned / local element layers (global indices)
  lorpc_mesh* m = nullptr;
  lorpc_lor* lor = nullptr;
  lorpc_prec* prec = nullptr;
  long long plane = 0;                 // nodes per z-plane
  long long own0 = 0, nown = 0;        // owned nodes: local offset and count
  long long gown0 = 0;                 // global index of the first owned node
  int vown0 = 0, nvown = 0;            // owned vertex planes: local index and count
  double *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr, *tmp = nullptr;
  double *part = nullptr, *Sl = nullptr, *Sg = nullptr, *hp = nullptr;
  double* rc = nullptr;                // global coarse residual (NCCL mode: own copy; emulation: shared)
};

struct lorpc_dist {
  int nranks = 1, nlocal = 1;
  bool emul = true;
  ncclComm_t comm = nullptr;
  int d = 3, p = 1, n[3] = {0, 0, 0};
  long long gplane = 0, gverts = 0;
  std::vector<DistRank> R;
  lorpc_prec* coarse = nullptr;        // replicated R_0 hierarchy on the global vertex grid
  lorpc_mesh* cmesh = nullptr;         // dims holder for the coarse object (no geometry)
  double* Ac0 = nullptr;               // global vertex-level operator (gathered)
  double* rc_shared = nullptr;         // emulation: the one global coarse vector
  double** d_loc = nullptr;            // emulation: device arrays of the ranks' scalar pointers
  double** d_glob = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace {

int nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) return fail(LORPC_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
  return LORPC_OK;
}
#define LORPC_NCCL(call) LORPC_TRY(nccl_check((call), #call))

// Exchange phases of one rank (local plane indices; -1 = none).  Phase k of rank
// r sends nplanes planes from send0 to rank `to` and receives nplanes planes into
// recv0 from rank `from` (overwritten for E1/E3, accumulated on free nodes for
// E2/E4).
int plan_of(int nz, int p, int R, int r, lorpc_dist_plan* P) {
  if (R < 1 || r < 0 || r >= R || nz < R || p < 1) return fail(LORPC_ERR_ARG, "dist plan: need nz >= nranks >= 1, p >= 1");
  memset(P, 0, sizeof(*P));
  P->z0 = (int)((long long)nz * r / R);
  P->z1 = (int)((long long)nz * (r + 1) / R);
  P->za = std::max(P->z0 - 1, 0);
  P->zb = std::min(P->z1 + 1, nz);
  P->own_plane0 = (P->z0 - P->za) * p;
  P->own_planes = (P->z1 - P->z0) * p + (r == R - 1 ? 1 : 0);
  P->gown_plane0 = P->z0 * p;
  P->vown0 = P->z0 - P->za;
  P->nvown = P->z1 - P->z0 + (r == R - 1 ? 1 : 0);
  const bool up = r + 1 < R, down = r > 0;
  for (int k = 0; k < 4; ++k) { P->to[k] = P->from[k] = -1; P->send0[k] = P->recv0[k] = -1; }
  P->nplanes[0] = P->nplanes[1] = 1;
  P->nplanes[2] = P->nplanes[3] = p - 1;
  // E1 operator input: own bottom plane z0 p down, plane z1 p from above
  if (down) { P->to[0] = r - 1; P->send0[0] = (P->z0 - P->za) * p; }
  if (up) { P->from[0] = r + 1; P->recv0[0] = (P->z1 - P->za) * p; }
  // E2 operator output: partial sums of plane z1 p up, added into plane z0 p
  if (up) { P->to[1] = r + 1; P->send0[1] = (P->z1 - P->za) * p; }
  if (down) { P->from[1] = r - 1; P->recv0[1] = (P->z0 - P->za) * p; }
  if (p >= 2) {
    // E3 Schwarz input: top p-1 owned planes up, the p-1 planes below z0 p from below
    if (up) { P->to[2] = r + 1; P->send0[2] = (P->z1 - 1 - P->za) * p + 1; }
    if (down) { P->from[2] = r - 1; P->recv0[2] = (P->z0 - 1 - P->za) * p + 1; }
    // E4 Schwarz output: patch sums on those planes down, added into the top planes
    if (down) { P->to[3] = r - 1; P->send0[3] = (P->z0 - 1 - P->za) * p + 1; }
    if (up) { P->from[3] = r + 1; P->recv0[3] = (P->z1 - 1 - P->za) * p + 1; }
  }
  return LORPC_OK;
}

// phase k (0..3) of the exchange on vector v of every local rank
int exchange(lorpc_dist* D, int k, double* DistRank::*v) {
  const bool add = k == 1 || k == 3;
  const int Nx = D->R[0].m->N[0], Ny = D->R[0].m->N[1];
  const long long pl = D->gplane;
  if (D->emul) {
    for (DistRank& S : D->R) {
      if (S.plan.to[k] < 0) continue;
      DistRank& T = D->R[S.plan.to[k]];
      const long long cnt = pl * S.plan.nplanes[k];
      const double* src = S.*v + S.plan.send0[k] * pl;
      double* dst = T.*v + T.plan.recv0[k] * pl;
      if (cnt == 0) continue;
      if (!add) {
        LORPC_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * cnt, cudaMemcpyDeviceToDevice, D->s));
      } else {
        k_add_planes_free<<<nb(cnt, 256), 256, 0, D->s>>>(dst, src, Nx, Ny, cnt);
        LORPC_LAUNCHED();
      }
    }
    return LORPC_OK;
  }
  DistRank& R = D->R[0];
  const long long cnt = pl * R.plan.nplanes[k];
  if (cnt == 0) return LORPC_OK;
  double* rbuf = add ? R.tmp : R.*v + R.plan.recv0[k] * pl;
  LORPC_NCCL(ncclGroupStart());
  // the group is closed before any error is returned (an open group would leave the
  // communicator unusable)
  ncclResult_t e1 = ncclSuccess, e2 = ncclSuccess;
  if (R.plan.to[k] >= 0) e1 = ncclSend(R.*v + R.plan.send0[k] * pl, (size_t)cnt, ncclDouble, R.plan.to[k], D->comm, D->s);
  if (e1 == ncclSuccess && R.plan.from[k] >= 0) e2 = ncclRecv(rbuf, (size_t)cnt, ncclDouble, R.plan.from[k], D->comm, D->s);
  const ncclResult_t e3 = ncclGroupEnd();
  LORPC_NCCL(e1);
  LORPC_NCCL(e2);
  LORPC_NCCL(e3);
  if (add && R.plan.from[k] >= 0) {
    k_add_planes_free<<<nb(cnt, 256), 256, 0, D->s>>>(R.*v + R.plan.recv0[k] * pl, rbuf, Nx, Ny, cnt);
    LORPC_LAUNCHED();
  }
  return LORPC_OK;
}

// global sum of scalar slot k (local values Sl[k] -> Sg[k] on every rank)
int allreduce_scalar(lorpc_dist* D, int k) {
  if (D->emul) {
    k_rank_sum<<<1, 1, 0, D->s>>>(D->d_loc, D->d_glob, D->nlocal, k);
    LORPC_LAUNCHED();
    return LORPC_OK;
  }
  LORPC_NCCL(ncclAllReduce(D->R[0].Sl + k, D->R[0].Sg + k, 1, ncclDouble, ncclSum, D->comm, D->s));
  return LORPC_OK;
}
// local owned dot a.b -> Sl[k] of every local rank, then the global sum
int ddot(lorpc_dist* D, double* DistRank::*a, double* DistRank::*b, int k) {
  for (DistRank& R : D->R) {
    k_ddot<<<DRED_BLOCKS, DRED_THREADS, 0, D->s>>>(R.*a + R.own0, R.*b + R.own0, R.nown, R.part);
    LORPC_LAUNCHED();
    k_dsum<<<1, 512, 0, D->s>>>(R.part, DRED_BLOCKS, R.Sl + k);
    LORPC_LAUNCHED();
  }
  return allreduce_scalar(D, k);
}

// q = A p on the owned nodes (E1, local element-layer apply, E2)
int dist_operator(lorpc_dist* D) {
  LORPC_TRY(exchange(D, 0, &DistRank::p));
  for (DistRank& R : D->R) LORPC_TRY(cg_apply(R.m, R.p, R.q, D->s));
  return exchange(D, 1, &DistRank::q);
}

// z = B r on the owned nodes: E3, patches, E4, coarse term
int dist_precond(lorpc_dist* D) {
  LORPC_TRY(exchange(D, 2, &DistRank::r));
  for (DistRank& R : D->R) LORPC_TRY(schwarz_apply_patches(R.prec, R.r, R.z, D->s));
  LORPC_TRY(exchange(D, 3, &DistRank::z));
  // coarse residual on the global vertex grid: each rank its owned vertex planes
  const long long gv = D->gverts;
  if (!D->emul) LORPC_CUDA(cudaMemsetAsync(D->R[0].rc, 0, sizeof(double) * gv, D->s));
  for (DistRank& R : D->R) {
    const lorpc_mesh* m = R.m;
    int3 nv = make_int3(m->n[0] + 1, m->n[1] + 1, m->n[2] + 1), N = make_int3(m->N[0], m->N[1], m->N[2]);
    const long long per = (long long)nv.x * nv.y;
    double* rcl = R.rc + per * R.za;  // local vertex plane k -> global plane za + k
    k_restrict_vertex_planes<<<nb(per * R.nvown, 128), 128, 0, D->s>>>(R.r, rcl, nv, N, m->basis, R.vown0,
                                                                      R.vown0 + R.nvown, R.za, D->n[2] + 1);
    LORPC_LAUNCHED();
  }
  if (!D->emul)
    LORPC_NCCL(ncclAllReduce(D->R[0].rc, D->coarse->cr[0], (size_t)gv, ncclDouble, ncclSum, D->comm, D->s));
  else
    LORPC_CUDA(cudaMemcpyAsync(D->coarse->cr[0], D->rc_shared, sizeof(double) * gv, cudaMemcpyDeviceToDevice, D->s));
  const double* zc = nullptr;
  LORPC_TRY(gmg_vcycle(D->coarse, &zc, D->s));
  for (DistRank& R : D->R)
    LORPC_TRY(prolong_vertex_add(R.m, zc + (long long)(R.m->n[0] + 1) * (R.m->n[1] + 1) * R.za, R.z, D->s));
  return LORPC_OK;
}

void destroy_rank(DistRank& R) {
  if (R.prec) lorpc_prec_destroy(R.prec);
  if (R.lor) lorpc_lor_destroy(R.lor);
  if (R.m) lorpc_mesh_destroy(R.m);
  dfree(R.x); dfree(R.r); dfree(R.z); dfree(R.p); dfree(R.q); dfree(R.tmp);
  dfree(R.part); dfree(R.Sl); dfree(R.Sg);
  if (R.hp) cudaFreeHost(R.hp);
  R.hp = nullptr; R.prec = nullptr; R.lor = nullptr; R.m = nullptr;
}

}  // namespace

extern "C" {

int lorpc_dist_plan_get(int nz, int p, int nranks, int rank, lorpc_dist_plan* out) {
  if (!out) return fail(LORPC_ERR_ARG, "dist_plan_get: NULL");
  return plan_of(nz, p, nranks, rank, out);
}

int lorpc_dist_nccl_id(void* id128) {
  if (!id128) return fail(LORPC_ERR_ARG, "dist_nccl_id: NULL");
  ncclUniqueId id;
  LORPC_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  memcpy(id128, &id, sizeof(id));
  return LORPC_OK;
}

void lorpc_dist_destroy(lorpc_dist* D) {
  if (!D) return;
  for (DistRank& R : D->R) destroy_rank(R);
  if (D->coarse) {
    lorpc_prec* c = D->coarse;
    for (int l = 1; l < c->nc; ++l) dfree(c->Ac[l]);
    for (int l = 0; l < c->nc; ++l) { dfree(c->dl1[l]); dfree(c->cr[l]); dfree(c->cz[l]); dfree(c->cs[l]); }
    dfree(c->coarse_chol); dfree(c->coarse_idx);
    delete c;
  }
  delete D->cmesh;
  dfree(D->Ac0);
  dfree(D->rc_shared);
  if (D->d_loc) cudaFree(D->d_loc);
  if (D->d_glob) cudaFree(D->d_glob);
  if (D->comm) ncclCommDestroy(D->comm);
  if (D->ev0) cudaEventDestroy(D->ev0);
  if (D->ev1) cudaEventDestroy(D->ev1);
  delete D;
}

int lorpc_dist_create(const lorpc_mesh_desc* desc, const double* vertices_host, const lorpc_schwarz_desc* sdesc,
                      int nranks, int rank, const void* nccl_id, void* stream, lorpc_dist** out) {
  if (!desc || !vertices_host || !sdesc || !out) return fail(LORPC_ERR_ARG, "dist_create: NULL argument");
  *out = nullptr;
  if (desc->dim != 3 || desc->disc != 0) return fail(LORPC_ERR_SIZE, "dist_create: 3D CG only");
  if (sdesc->patch_kind != 0 || sdesc->coarse != 0)
    return fail(LORPC_ERR_SIZE, "dist_create: vertex patches with the GMG coarse term only");
  if (nranks < 1 || desc->n[2] < nranks) return fail(LORPC_ERR_ARG, "dist_create: need n_z >= nranks >= 1");
  if (nccl_id && (rank < 0 || rank >= nranks)) return fail(LORPC_ERR_ARG, "dist_create: bad rank");
  lorpc_dist* D = new lorpc_dist();
  D->nranks = nranks;
  D->emul = nccl_id == nullptr;
  D->nlocal = D->emul ? nranks : 1;
  D->d = 3; D->p = desc->p;
  for (int k = 0; k < 3; ++k) D->n[k] = desc->n[k];
  D->s = (cudaStream_t)stream;
  const long long nvx = desc->n[0] + 1, nvy = desc->n[1] + 1, nvz = desc->n[2] + 1;
  D->gplane = (long long)(desc->n[0] * desc->p + 1) * (desc->n[1] * desc->p + 1);
  D->gverts = nvx * nvy * nvz;
  auto bail = [&](int rc) { lorpc_dist_destroy(D); return rc; };
  if (!D->emul) {
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    int rc = nccl_check(ncclCommInitRank(&D->comm, nranks, id, rank), "ncclCommInitRank");
    if (rc != LORPC_OK) return bail(rc);
  }
  D->R.resize((size_t)D->nlocal);
  for (int i = 0; i < D->nlocal; ++i) {
    DistRank& R = D->R[i];
    R.rank = D->emul ? i : rank;
    int rc = plan_of(desc->n[2], desc->p, nranks, R.rank, &R.plan);
    if (rc != LORPC_OK) return bail(rc);
    R.z0 = R.plan.z0; R.z1 = R.plan.z1; R.za = R.plan.za; R.zb = R.plan.zb;
    lorpc_mesh_desc ld = *desc;
    ld.n[2] = R.zb - R.za;
    const double* vl = vertices_host + (size_t)(nvx * nvy * R.za) * 3;
    rc = lorpc_mesh_create(&ld, vl, stream, &R.m);
    if (rc != LORPC_OK) return bail(rc);
    R.m->ez_lo = R.z0 - R.za;
    R.m->ez_hi = R.z1 - R.za;
    rc = lorpc_lor_assemble(R.m, stream, &R.lor);
    if (rc != LORPC_OK) return bail(rc);
    // patches of the owned vertex planes, no coarse term (R_0 is global below)
    R.vown0 = R.plan.vown0;
    R.nvown = R.plan.nvown;
    {
      lorpc_prec* b = new lorpc_prec();
      b->lor = R.lor; b->m = R.m; b->desc = *sdesc; b->desc.coarse = 1;
      b->pvz0 = R.vown0; b->pnvz = R.nvown;
      R.prec = b;
      rc = schwarz_build(b, (cudaStream_t)stream);
      if (rc != LORPC_OK) return bail(rc);
    }
    R.plane = D->gplane;
    R.own0 = (long long)R.plan.own_plane0 * R.plane;
    R.nown = (long long)R.plan.own_planes * R.plane;
    R.gown0 = (long long)R.plan.gown_plane0 * R.plane;
    const long long nl = R.m->ndof_cg;
    if ((rc = dalloc(&R.x, (size_t)nl)) || (rc = dalloc(&R.r, (size_t)nl)) || (rc = dalloc(&R.z, (size_t)nl)) ||
        (rc = dalloc(&R.p, (size_t)nl)) || (rc = dalloc(&R.q, (size_t)nl)) ||
        (rc = dalloc(&R.tmp, (size_t)(2 * D->gplane * std::max(desc->p, 1)))) ||
        (rc = dalloc(&R.part, DRED_BLOCKS)) || (rc = dalloc(&R.Sl, D_NS)) || (rc = dalloc(&R.Sg, D_NS)))
      return bail(rc);
    for (double* v : {R.x, R.r, R.z, R.p, R.q})
      if (cudaMemsetAsync(v, 0, sizeof(double) * nl, D->s) != cudaSuccess) return bail(fail(LORPC_ERR_CUDA, "memset"));
    if (cudaMallocHost(&R.hp, sizeof(double) * D_NS) != cudaSuccess) return bail(fail(LORPC_ERR_OOM, "pinned"));
  }
  // coarse space: gather the owned vertex-plane rows of the last LOR level into the
  // global vertex operator A_0 (reading r1), then the replicated GMG hierarchy
  const int NDP = ndp_of(3);
  const long long per = nvx * nvy;
  int rc = dalloc(&D->Ac0, (size_t)(D->gverts * NDP));
  if (rc != LORPC_OK) return bail(rc);
  if (cudaMemsetAsync(D->Ac0, 0, sizeof(double) * D->gverts * NDP, D->s) != cudaSuccess)
    return bail(fail(LORPC_ERR_CUDA, "memset"));
  for (DistRank& R : D->R) {
    const double* src = R.lor->A[R.lor->L - 1] + (size_t)(per * R.vown0) * NDP;
    double* dst = D->Ac0 + (size_t)(per * R.z0) * NDP;
    if (cudaMemcpyAsync(dst, src, sizeof(double) * per * R.nvown * NDP, cudaMemcpyDeviceToDevice, D->s) != cudaSuccess)
      return bail(fail(LORPC_ERR_CUDA, "coarse gather copy"));
  }
  if (!D->emul) {
    rc = nccl_check(ncclAllReduce(D->Ac0, D->Ac0, (size_t)(D->gverts * NDP), ncclDouble, ncclSum, D->comm, D->s),
                    "ncclAllReduce(A_0)");
    if (rc != LORPC_OK) return bail(rc);
  }
  D->cmesh = new lorpc_mesh();
  D->cmesh->d = 3;
  D->coarse = new lorpc_prec();
  D->coarse->m = D->cmesh;
  const int nv[3] = {(int)nvx, (int)nvy, (int)nvz};
  rc = gmg_build(D->coarse, D->Ac0, nv, 3, D->s);
  if (rc != LORPC_OK) return bail(rc);
  if (D->emul) {
    if ((rc = dalloc(&D->rc_shared, (size_t)D->gverts)) != LORPC_OK) return bail(rc);
    cudaMemsetAsync(D->rc_shared, 0, sizeof(double) * D->gverts, D->s);
    for (DistRank& R : D->R) R.rc = D->rc_shared;
    std::vector<double*> hl, hg;
    for (DistRank& R : D->R) { hl.push_back(R.Sl); hg.push_back(R.Sg); }
    if (cudaMalloc(&D->d_loc, sizeof(double*) * hl.size()) != cudaSuccess ||
        cudaMalloc(&D->d_glob, sizeof(double*) * hg.size()) != cudaSuccess)
      return bail(fail(LORPC_ERR_OOM, "dist pointers"));
    cudaMemcpyAsync(D->d_loc, hl.data(), sizeof(double*) * hl.size(), cudaMemcpyHostToDevice, D->s);
    cudaMemcpyAsync(D->d_glob, hg.data(), sizeof(double*) * hg.size(), cudaMemcpyHostToDevice, D->s);
  } else {
    if ((rc = dalloc(&D->R[0].rc, (size_t)D->gverts)) != LORPC_OK) return bail(rc);
  }
  cudaEventCreate(&D->ev0);
  cudaEventCreate(&D->ev1);
  if (cudaStreamSynchronize(D->s) != cudaSuccess) return bail(fail(LORPC_ERR_CUDA, "dist_create sync"));
  *out = D;
  return LORPC_OK;
}

int lorpc_dist_info(const lorpc_dist* D, int local, long long* owned_offset, long long* n_owned, long long* n_patches) {
  if (!D || local < 0 || local >= D->nlocal) return fail(LORPC_ERR_ARG, "dist_info: bad handle/local rank");
  const DistRank& R = D->R[local];
  if (owned_offset) *owned_offset = R.gown0;
  if (n_owned) *n_owned = R.nown;
  if (n_patches) *n_patches = R.prec->J;
  return LORPC_OK;
}

int lorpc_dist_local_prec(const lorpc_dist* D, int local, const lorpc_prec** out) {
  if (!D || !out || local < 0 || local >= D->nlocal) return fail(LORPC_ERR_ARG, "dist_local_prec: bad argument");
  *out = D->R[local].prec;
  return LORPC_OK;
}

int lorpc_dist_operator_apply(lorpc_dist* D, const double* const* x_owned, double* const* y_owned) {
  if (!D || !x_owned || !y_owned) return fail(LORPC_ERR_ARG, "dist_operator_apply: NULL");
  for (int i = 0; i < D->nlocal; ++i)
    LORPC_CUDA(cudaMemcpyAsync(D->R[i].p + D->R[i].own0, x_owned[i], sizeof(double) * D->R[i].nown,
                               cudaMemcpyDeviceToDevice, D->s));
  LORPC_TRY(dist_operator(D));
  for (int i = 0; i < D->nlocal; ++i)
    LORPC_CUDA(cudaMemcpyAsync(y_owned[i], D->R[i].q + D->R[i].own0, sizeof(double) * D->R[i].nown,
                               cudaMemcpyDeviceToDevice, D->s));
  return LORPC_OK;
}

int lorpc_dist_precond_apply(lorpc_dist* D, const double* const* r_owned, double* const* z_owned) {
  if (!D || !r_owned || !z_owned) return fail(LORPC_ERR_ARG, "dist_precond_apply: NULL");
  for (int i = 0; i < D->nlocal; ++i)
    LORPC_CUDA(cudaMemcpyAsync(D->R[i].r + D->R[i].own0, r_owned[i], sizeof(double) * D->R[i].nown,
                               cudaMemcpyDeviceToDevice, D->s));
  LORPC_TRY(dist_precond(D));
  for (int i = 0; i < D->nlocal; ++i)
    LORPC_CUDA(cudaMemcpyAsync(z_owned[i], D->R[i].z + D->R[i].own0, sizeof(double) * D->R[i].nown,
                               cudaMemcpyDeviceToDevice, D->s));
  return LORPC_OK;
}

int lorpc_dist_pcg_solve(lorpc_dist* D, const double* const* b_owned, double* const* x_owned, double rtol, int maxit,
                         lorpc_pcg_report* rep) {
  if (!D || !b_owned || !x_owned || !rep) return fail(LORPC_ERR_ARG, "dist_pcg_solve: NULL");
  cudaStream_t s = D->s;
  rep->iters = 0; rep->converged = 0; rep->rel_res = 1.0; rep->t_solve_ms = 0.0;
  LORPC_CUDA(cudaEventRecord(D->ev0, s));
  for (int i = 0; i < D->nlocal; ++i) {
    DistRank& R = D->R[i];
    LORPC_CUDA(cudaMemcpyAsync(R.r + R.own0, b_owned[i], sizeof(double) * R.nown, cudaMemcpyDeviceToDevice, s));
    LORPC_CUDA(cudaMemsetAsync(R.x + R.own0, 0, sizeof(double) * R.nown, s));
  }
  LORPC_TRY(ddot(D, &DistRank::r, &DistRank::r, D_BB));
  DistRank& R0 = D->R[0];
  LORPC_CUDA(cudaMemcpyAsync(R0.hp, R0.Sg, sizeof(double) * D_NS, cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  const double nb2 = std::sqrt(R0.hp[D_BB]);
  if (rep->res_hist) rep->res_hist[0] = 1.0;
  if (nb2 == 0.0) {
    rep->converged = 1; rep->rel_res = 0.0;
    for (int i = 0; i < D->nlocal; ++i) LORPC_CUDA(cudaMemsetAsync(x_owned[i], 0, sizeof(double) * D->R[i].nown, s));
    return LORPC_OK;
  }
  LORPC_TRY(dist_precond(D));
  for (DistRank& R : D->R)
    LORPC_CUDA(cudaMemcpyAsync(R.p + R.own0, R.z + R.own0, sizeof(double) * R.nown, cudaMemcpyDeviceToDevice, s));
  LORPC_TRY(ddot(D, &DistRank::r, &DistRank::z, D_RHO));
  int status = LORPC_ERR_NOT_CONVERGED;
  double rho_prev = 0.0;
  for (int k = 1; k <= maxit; ++k) {
    LORPC_TRY(dist_operator(D));
    LORPC_TRY(ddot(D, &DistRank::p, &DistRank::q, D_PQ));
    for (DistRank& R : D->R) {
      k_dupdate_xr<<<DRED_BLOCKS, DRED_THREADS, 0, s>>>(R.x + R.own0, R.r + R.own0, R.p + R.own0, R.q + R.own0, R.nown,
                                                        R.Sg);
      LORPC_LAUNCHED();
    }
    LORPC_TRY(ddot(D, &DistRank::r, &DistRank::r, D_RR));
    LORPC_CUDA(cudaMemcpyAsync(R0.hp, R0.Sg, sizeof(double) * D_NS, cudaMemcpyDeviceToHost, s));
    LORPC_CUDA(cudaStreamSynchronize(s));
    rep->iters = k;
    const double alpha = R0.hp[D_RHO] / R0.hp[D_PQ];
    if (rep->alpha) rep->alpha[k - 1] = alpha;
    if (k >= 2 && rep->beta) rep->beta[k - 2] = R0.hp[D_RHO] / rho_prev;
    rho_prev = R0.hp[D_RHO];
    if (!(R0.hp[D_PQ] > 0.0)) {
      status = fail(LORPC_ERR_BREAKDOWN, "dist pcg: p.Ap <= 0 at iteration " + std::to_string(k));
      break;
    }
    const double rel = std::sqrt(R0.hp[D_RR]) / nb2;
    rep->rel_res = rel;
    if (rep->res_hist) rep->res_hist[k] = rel;
    if (rel <= rtol) { rep->converged = 1; status = LORPC_OK; break; }
    LORPC_TRY(dist_precond(D));
    LORPC_TRY(ddot(D, &DistRank::r, &DistRank::z, D_RZ));
    for (DistRank& R : D->R) {
      k_dupdate_p<<<DRED_BLOCKS, DRED_THREADS, 0, s>>>(R.p + R.own0, R.z + R.own0, R.nown, R.Sg);
      LORPC_LAUNCHED();
      k_dset<<<1, 1, 0, s>>>(R.Sg, D_RHO, D_RZ);
      LORPC_LAUNCHED();
    }
  }
  for (int i = 0; i < D->nlocal; ++i)
    LORPC_CUDA(cudaMemcpyAsync(x_owned[i], D->R[i].x + D->R[i].own0, sizeof(double) * D->R[i].nown,
                               cudaMemcpyDeviceToDevice, s));
  LORPC_CUDA(cudaEventRecord(D->ev1, s));
  LORPC_CUDA(cudaEventSynchronize(D->ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, D->ev0, D->ev1);
  rep->t_solve_ms = ms;
  if (status == LORPC_ERR_NOT_CONVERGED) return fail(status, "dist pcg: not converged in " + std::to_string(maxit));
  return status;
}

}  // extern "C"
