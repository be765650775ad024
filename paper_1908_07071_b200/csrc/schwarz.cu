// Additive Schwarz preconditioner B = sum_j R_j Q_j + P_0 R_0 P_0^T (eq:as
// P:274-277), rows a5-a8 and a11 of the hot-path table.
//
// Setup (k_mdf_ilu): one warp per (patch, level).  The patch operator A_j at
// level l is the global level-l stencil restricted to the patch's free node
// box (reading c4).  The warp runs the minimum-discarded-fill ordering fused
// with the ILU(0) elimination on the fixed 3^d pattern (reading c6: weight
// w_k^2 = sum over non-pattern pairs of (A_ik A_kj / A_kk)^2, minimum of
// (q30(w^2), index)), giving M = L D L^T (reading c5); then the DAG level
// schedule of the triangular solves.  Arithmetic of the weights and of the
// elimination update uses explicit round-to-nearest intrinsics (no FMA
// contraction) so that the ordering decisions match a plain evaluation.
//
// Apply (k_vcycle): one warp per patch, patch vectors of every level in shared
// memory; V(1,1) with one ILU(0) smoothing step before and after
// (level-scheduled forward / backward solves), residuals with the global level
// stencils, restriction / prolongation by the GLL reference-coordinate
// weights, exact LDL^T at the coarsest level (reading c8); the patch result is
// added into z with atomics (a8).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "patch.cuh"

namespace lorpc {

int galerkin(int d, const double* Af, double* Ac, const Transfer1D& T, const int* ne, const int* Nf, const int* Nc,
             cudaStream_t s);
Transfer1D gmg_transfer();
int dense_coarse_setup(lorpc_prec* b, cudaStream_t s);  // vcycle.cu
int trec_build(lorpc_prec* b, cudaStream_t s);          // vcycle_t.cu
size_t tmode_smem(const lorpc_prec* b);
int wrec_build(lorpc_prec* b, cudaStream_t s);          // vcycle_w.cu
int single_setup(lorpc_prec* b);                        // single.cu
size_t wmode_smem(const lorpc_prec* b);
int qrec_build(lorpc_prec* b, cudaStream_t s, int* ok);  // vcycle_w.cu (Q mode)
size_t qmode_smem(const lorpc_prec* b);

// ------------------------------------------------------------------ MDF + ILU(0)
__device__ __forceinline__ double q30(double x) {
  if (x == 0.0) return 0.0;
  int e;
  const double f = frexp(x, &e);
  return ldexp(rint(ldexp(f, 30)), e - 30);
}

__device__ __forceinline__ bool adjacent(int di, int dj) {
  return abs(dir_dx(di) - dir_dx(dj)) <= 1 && abs(dir_dy(di) - dir_dy(dj)) <= 1 && abs(dir_dz(di) - dir_dz(dj)) <= 1;
}
// direction index from i to j given the offsets of i and j from k
template <int DIM>
__device__ __forceinline__ int dir_between(int di, int dj) {
  int r = (dir_dx(dj) - dir_dx(di) + 1) + 3 * (dir_dy(dj) - dir_dy(di) + 1);
  if (DIM == 3) r += 9 * (dir_dz(dj) - dir_dz(di) + 1);
  return r;
}

template <int DIM>
__device__ double mdf_w2(const double* At, const unsigned char* alive, int m, uint32_t em, int ex, int ey) {
  constexpr int ND = Dirs<DIM>::ND, C = Dirs<DIM>::CENTER;
  const double amm = At[m * ND + C];
  double s = 0.0;
  for (int di = 0; di < ND; ++di) {
    if (di == C || !((em >> di) & 1u)) continue;
    if (!alive[m + doff<DIM>(di, ex, ey)]) continue;
    for (int dj = 0; dj < ND; ++dj) {
      if (dj == C || dj == di || !((em >> dj) & 1u)) continue;
      if (!alive[m + doff<DIM>(dj, ex, ey)]) continue;
      if (adjacent(di, dj)) continue;
      const double f = __ddiv_rn(__dmul_rn(At[m * ND + di], At[m * ND + dj]), amm);
      s = __dadd_rn(s, __dmul_rn(f, f));
    }
  }
  return s;
}

struct MdfParams {
  PatchGeom G;
  const double* A[MAXL];
  char* rec;
  const long long* recoff;
  long long ntasks;     // J * L
  int ordering;
  int maxn;
  double* scratch;      // per warp: At[maxn*ND], Lf[maxn*ND], w2[maxn]
  int* iscratch;        // per warp: pos, lev, order, cnt(+1), lmask [maxn]; pmap [maxn*ND]
  unsigned char* alive; // per warp: maxn
  unsigned long long* err;  // first failing task (patch*L + level) or ~0
  int* err_step;
};

template <int DIM>
__global__ void __launch_bounds__(128) k_mdf_ilu(MdfParams P) {
  constexpr int ND = Dirs<DIM>::ND, C = Dirs<DIM>::CENTER;
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  double* At = P.scratch + gw * (long long)P.maxn * (2 * ND + 1);
  double* Lf = At + (long long)P.maxn * ND;
  double* w2 = Lf + (long long)P.maxn * ND;
  int* pos = P.iscratch + gw * (long long)((5 + ND) * P.maxn + 1);
  int* lev = pos + P.maxn;
  int* ord = lev + P.maxn;
  int* cnt = ord + P.maxn;
  int* lmk = cnt + P.maxn + 1;
  int* pmap = lmk + P.maxn;
  unsigned char* alive = P.alive + gw * (long long)P.maxn;
  for (long long task = gw; task < P.ntasks; task += nw) {
    const long long j = task / P.G.L;
    const int l = (int)(task % P.G.L);
    int lo[3], ext[3];
    patch_box(P.G, j, l, lo, ext);
    const int ex = ext[0], ey = ext[1], ez = ext[2];
    const int n = ex * ey * ez;
    char* rec = P.rec + P.recoff[task];
    const long long nL = num_edges(DIM, ext);
    const RecLayout R = rec_layout(n, nL);
    if (n <= 0) {
      if (lane == 0) { int* h = (int*)rec; h[0] = 0; h[1] = 0; h[2] = 0; h[3] = l; }
      continue;
    }
    const long long Nx = P.G.Nax[l][0], Ny = P.G.Nax[l][1];
    const double* A = P.A[l];
    for (int i = lane; i < n; i += 32) {
      const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
      const long long gi = (lo[0] + ix) + Nx * ((lo[1] + iy) + Ny * (DIM == 3 ? lo[2] + iz : 0));
      const uint32_t em = exist_mask<DIM>(ix, iy, iz, ex, ey, ez);
      for (int d = 0; d < ND; ++d) {
        At[i * ND + d] = ((em >> d) & 1u) ? A[gi * Dirs<DIM>::NDP + d] : 0.0;
        Lf[i * ND + d] = 0.0;
      }
      alive[i] = 1;
      pos[i] = -1;
    }
    __syncwarp();
    if (P.ordering == 0)
      for (int i = lane; i < n; i += 32) {
        const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
        w2[i] = mdf_w2<DIM>(At, alive, i, exist_mask<DIM>(ix, iy, iz, ex, ey, ez), ex, ey);
      }
    if (P.ordering == 2 && lane == 0) {
      // reverse Cuthill-McKee on the box's 3^d-stencil graph (structure only; reading
      // r5: minimum-degree start, lowest index on ties, neighbours by (degree, index),
      // reversed), into lev[] (free until the DAG levels are formed); cnt[] = queue,
      // pos[] = visited marks (reset below)
      int* q = cnt;
      int tail = 0, head = 0;
      while (tail < n) {
        int s0 = -1, ds = 99;
        for (int i = 0; i < n; ++i) {
          if (pos[i] != -1) continue;
          const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
          const int dg = __popc(exist_mask<DIM>(ix, iy, iz, ex, ey, ez)) - 1;
          if (dg < ds) { ds = dg; s0 = i; }
        }
        pos[s0] = -2;
        q[tail++] = s0;
        while (head < tail) {
          const int v = q[head++];
          const int vx = v % ex, vy = (v / ex) % ey, vz = v / (ex * ey);
          const uint32_t ev = exist_mask<DIM>(vx, vy, vz, ex, ey, ez);
          const int t0 = tail;
          for (int dd = 0; dd < ND; ++dd) {
            if (dd == C || !((ev >> dd) & 1u)) continue;
            const int u = v + doff<DIM>(dd, ex, ey);
            if (pos[u] != -1) continue;
            pos[u] = -2;
            // insertion by (degree, index)
            const int ux = u % ex, uy = (u / ex) % ey, uz = u / (ex * ey);
            const int du = __popc(exist_mask<DIM>(ux, uy, uz, ex, ey, ez)) - 1;
            int t = tail++;
            while (t > t0) {
              const int w = q[t - 1];
              const int wx = w % ex, wy = (w / ex) % ey, wz = w / (ex * ey);
              const int dw = __popc(exist_mask<DIM>(wx, wy, wz, ex, ey, ez)) - 1;
              if (dw < du || (dw == du && w < u)) break;
              q[t] = w;
              --t;
            }
            q[t] = u;
          }
        }
      }
      for (int t = 0; t < n; ++t) { lev[t] = q[n - 1 - t]; pos[t] = -1; }
    }
    __syncwarp();
    bool failed = false;
    for (int step = 0; step < n; ++step) {
      double bk = INFINITY;
      int bi = 0x7fffffff;
      if (P.ordering == 2) {
        bi = lev[step];
      } else {
        for (int i = lane; i < n; i += 32) {
          if (!alive[i]) continue;
          const double key = P.ordering == 0 ? q30(w2[i]) : 0.0;
          if (key < bk || (key == bk && i < bi)) { bk = key; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ok < bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
        }
      }
      const int k = bi;
      const int kx = k % ex, ky = (k / ex) % ey, kz = k / (ex * ey);
      const uint32_t ek = exist_mask<DIM>(kx, ky, kz, ex, ey, ez);
      const double akk = At[k * ND + C];
      if (!(akk > 0.0)) {
        if (lane == 0) {
          if (atomicCAS(P.err, ~0ull, (unsigned long long)task) == ~0ull) *P.err_step = step;
        }
        failed = true;
        break;
      }
      if (lane == 0) { ord[step] = k; pos[k] = step; }
      // L_ik = At_ik / At_kk for alive neighbours i (stored at (i, dir i->k))
      for (int di = lane; di < ND; di += 32) {
        if (di == C || !((ek >> di) & 1u)) continue;
        const int i = k + doff<DIM>(di, ex, ey);
        if (!alive[i]) continue;
        const int dik = ND - 1 - di;
        Lf[i * ND + dik] = __ddiv_rn(At[i * ND + dik], akk);
      }
      __syncwarp();
      // ILU(0) update on the pattern: At_ij -= (At_ki At_kj) / At_kk
      for (int pr = lane; pr < ND * ND; pr += 32) {
        const int di = pr / ND, dj = pr % ND;
        if (di == C || dj == C || !((ek >> di) & 1u) || !((ek >> dj) & 1u)) continue;
        if (!adjacent(di, dj)) continue;
        const int i = k + doff<DIM>(di, ex, ey), jj = k + doff<DIM>(dj, ex, ey);
        if (!alive[i] || !alive[jj]) continue;
        const int dij = dir_between<DIM>(di, dj);
        At[i * ND + dij] = __dsub_rn(At[i * ND + dij], __ddiv_rn(__dmul_rn(At[k * ND + di], At[k * ND + dj]), akk));
      }
      __syncwarp();
      if (lane == 0) alive[k] = 0;
      __syncwarp();
      if (P.ordering == 0) {
        for (int di = lane; di < ND; di += 32) {
          if (di == C || !((ek >> di) & 1u)) continue;
          const int i = k + doff<DIM>(di, ex, ey);
          if (!alive[i]) continue;
          const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
          w2[i] = mdf_w2<DIM>(At, alive, i, exist_mask<DIM>(ix, iy, iz, ex, ey, ez), ex, ey);
        }
      }
      __syncwarp();
    }
    if (failed) continue;
    // ---- record (layout: rec_layout in patch.cuh)
    double* Dr = (double*)(rec + R.D);
    double* Lr = (double*)(rec + R.L);
    uint16_t* nbr = (uint16_t*)(rec + R.nb);
    uint16_t* frp = (uint16_t*)(rec + R.frp);
    uint16_t* lpt = (uint16_t*)(rec + R.lptr);
    uint16_t* sch = (uint16_t*)(rec + R.sched);
    uint16_t* orr = (uint16_t*)(rec + R.order);
    for (int i = lane; i < n; i += 32) {
      Dr[i] = At[i * ND + C];  // pivot at elimination time (never modified afterwards)
      orr[i] = (uint16_t)ord[i];
      const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
      const uint32_t em = exist_mask<DIM>(ix, iy, iz, ex, ey, ez);
      uint32_t lm = 0;
      for (int d = 0; d < ND; ++d) {
        if (d == C || !((em >> d) & 1u)) continue;
        if (pos[i + doff<DIM>(d, ex, ey)] < pos[i]) lm |= 1u << d;
      }
      lmk[i] = (int)lm;
    }
    __syncwarp();
    if (lane == 0) {
      // DAG levels in elimination order
      int depth = 0;
      for (int i = 0; i < n; ++i) cnt[i] = 0;
      for (int t = 0; t < n; ++t) {
        const int i = ord[t];
        int lv = 0;
        uint32_t lm = (uint32_t)lmk[i];
        while (lm) {
          const int d = __ffs(lm) - 1;
          lm &= lm - 1;
          lv = max(lv, lev[i + doff<DIM>(d, ex, ey)] + 1);
        }
        lev[i] = lv;
        depth = max(depth, lv + 1);
        cnt[lv]++;
      }
      // level pointers + stable placement in elimination order
      int acc = 0;
      for (int v = 0; v < depth; ++v) { lpt[v] = (uint16_t)acc; const int c = cnt[v]; cnt[v] = acc; acc += c; }
      lpt[depth] = (uint16_t)acc;
      for (int t = 0; t < n; ++t) { const int i = ord[t]; sch[cnt[lev[i]]++] = (uint16_t)i; }
      // forward entries: rows in schedule order, each row's lower neighbours by direction
      int e = 0;
      for (int t = 0; t < n; ++t) {
        const int i = sch[t];
        frp[t] = (uint16_t)e;
        uint32_t lm = (uint32_t)lmk[i];
        while (lm) {
          const int d = __ffs(lm) - 1;
          lm &= lm - 1;
          Lr[e] = Lf[i * ND + d];
          nbr[e] = (uint16_t)(i + doff<DIM>(d, ex, ey));
          pmap[i * ND + d] = e;
          ++e;
        }
      }
      frp[n] = (uint16_t)e;
      // backward entries: row i pulls L_ki z_k from its later neighbours k
      uint16_t* bk = (uint16_t*)(rec + R.bk);
      double* bL = (double*)(rec + R.bL);
      uint16_t* brp = (uint16_t*)(rec + R.brp);
      int f = 0;
      for (int t = 0; t < n; ++t) {
        const int i = sch[t];
        brp[t] = (uint16_t)f;
        const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
        uint32_t um = exist_mask<DIM>(ix, iy, iz, ex, ey, ez) & ~(uint32_t)lmk[i] & ~(1u << C);
        while (um) {
          const int d = __ffs(um) - 1;
          um &= um - 1;
          const int k = i + doff<DIM>(d, ex, ey);
          bk[f] = (uint16_t)k;
          bL[f] = Lr[pmap[k * ND + (ND - 1 - d)]];
          ++f;
        }
      }
      brp[n] = (uint16_t)f;
      int* h = (int*)rec;
      h[0] = n; h[1] = depth; h[2] = (int)nL; h[3] = l;
    }
    __syncwarp();
  }
}


template <int DIM>
__global__ void k_l1diag(const double* __restrict__ A, double* __restrict__ dl, int3 Nv) {
  constexpr int ND = Dirs<DIM>::ND;
  const long long NT = (long long)Nv.x * Nv.y * Nv.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NT) return;
  const int c[3] = {(int)(g % Nv.x), (int)((g / Nv.x) % Nv.y), (int)(g / ((long long)Nv.x * Nv.y))};
  const int Nn[3] = {Nv.x, Nv.y, Nv.z};
  double s = 0.0;
  for (int d = 0; d < ND; ++d) {
    const int o[3] = {dir_dx(d), dir_dy(d), dir_dz(d)};
    bool in = true;
    for (int k = 0; k < DIM; ++k) { const int v = c[k] + o[k]; if (v <= 0 || v >= Nn[k] - 1) in = false; }
    if (in) s += fabs(A[g * Dirs<DIM>::NDP + d]);
  }
  dl[g] = s;
}

// GMG smoothing kernels on a vertex grid (interior nodes; boundary nodes hold 0)

// ------------------------------------------------------------------ setup driver
PatchGeom make_geom(const lorpc_prec* b) {
  PatchGeom G{};
  const lorpc_mesh* m = b->m;
  G.d = m->d; G.kind = b->desc.patch_kind; G.L = b->lor->L; G.vz0 = b->pvz0;
  G.erng = b->erng;
  for (int k = 0; k < 3; ++k) G.n[k] = m->n[k];
  for (int l = 0; l < G.L; ++l) {
    G.ml[l] = b->lor->ml[l];
    for (int k = 0; k < 3; ++k) G.Nax[l][k] = b->lor->Nax[l][k];
  }
  return G;
}

// R_0 hierarchy on a vertex grid nv (reading c11): level 0 operator Ac0 (full
// stencil, node-major; not owned), 2:1 Galerkin coarsening while every axis has
// an even number (> 2) of intervals, exact solve on the coarsest interior (any
// size up to 2048 vertices: odd or anisotropic grids stop coarsening early).
int gmg_build(lorpc_prec* b, double* Ac0, const int* nv, int d, cudaStream_t s) {
  b->nc = 0;
  for (int i = 0; i < MAXC; ++i) { b->Ac[i] = b->dl1[i] = b->cr[i] = b->cz[i] = b->cs[i] = nullptr; }
  int cur[3] = {nv[0], nv[1], d == 3 ? nv[2] : 1};
  b->Ac[0] = Ac0;
  int lvl = 0;
  while (true) {
    for (int k = 0; k < 3; ++k) b->cn[lvl][k] = cur[k];
    b->cN[lvl] = (long long)cur[0] * cur[1] * cur[2];
    LORPC_TRY(dalloc(&b->dl1[lvl], b->cN[lvl]));
    LORPC_TRY(dalloc(&b->cr[lvl], b->cN[lvl]));
    LORPC_TRY(dalloc(&b->cz[lvl], b->cN[lvl]));
    LORPC_TRY(dalloc(&b->cs[lvl], b->cN[lvl]));
    LORPC_CUDA(cudaMemsetAsync(b->cz[lvl], 0, sizeof(double) * b->cN[lvl], s));
    LORPC_CUDA(cudaMemsetAsync(b->cs[lvl], 0, sizeof(double) * b->cN[lvl], s));
    if (d == 2) k_l1diag<2><<<nb(b->cN[lvl], 256), 256, 0, s>>>(b->Ac[lvl], b->dl1[lvl], i3(cur));
    else k_l1diag<3><<<nb(b->cN[lvl], 256), 256, 0, s>>>(b->Ac[lvl], b->dl1[lvl], i3(cur));
    LORPC_LAUNCHED();
    bool can = true;
    for (int k = 0; k < d; ++k) if ((cur[k] - 1) % 2 != 0 || cur[k] - 1 <= 2) can = false;
    if (!can || lvl + 1 >= MAXC) break;
    int nxt[3] = {cur[0], cur[1], cur[2]};
    for (int k = 0; k < d; ++k) nxt[k] = (cur[k] - 1) / 2 + 1;
    long long Nn = (long long)nxt[0] * nxt[1] * nxt[2];
    LORPC_TRY(dalloc(&b->Ac[lvl + 1], (size_t)ndp_of(d) * Nn));
    int ne[3] = {nxt[0] - 1, nxt[1] - 1, nxt[2] - 1};
    LORPC_TRY(galerkin(d, b->Ac[lvl], b->Ac[lvl + 1], gmg_transfer(), ne, cur, nxt, s));
    for (int k = 0; k < 3; ++k) cur[k] = nxt[k];
    ++lvl;
  }
  b->nc = lvl + 1;
  // coarsest level: exact solve (reading c11) through the dense inverse of its interior
  // matrix, formed once here on the host (Cholesky, then L^{-T} L^{-1}); the apply is
  // a parallel dense matvec (k_coarsest_inv)
  const int3 nvl = i3(b->cn[lvl]);
  const long long NT = b->cN[lvl];
  std::vector<int> ilist;
  for (long long g = 0; g < NT; ++g) {
    const int c[3] = {(int)(g % nvl.x), (int)((g / nvl.x) % nvl.y), (int)(g / ((long long)nvl.x * nvl.y))};
    bool in = c[0] > 0 && c[0] < nvl.x - 1 && c[1] > 0 && c[1] < nvl.y - 1;
    if (d == 3) in = in && c[2] > 0 && c[2] < nvl.z - 1;
    if (in) ilist.push_back((int)g);
  }
  const int nint = (int)ilist.size();
  if (nint > 2048)
    return fail(LORPC_ERR_SIZE, "coarsest GMG level has " + std::to_string(nint) +
                                    " interior vertices (> 2048): the vertex grid does not halve evenly enough");
  b->ncoarsest = nint;
  LORPC_TRY(dalloc(&b->coarse_chol, (size_t)std::max(nint * nint, 1)));
  LORPC_TRY(dalloc(&b->coarse_idx, (size_t)std::max(nint, 1)));
  if (nint > 0) {
    const int ndp = ndp_of(d), ND = d == 2 ? 9 : 27;
    std::vector<double> A((size_t)NT * ndp);
    LORPC_CUDA(cudaMemcpyAsync(A.data(), b->Ac[lvl], sizeof(double) * A.size(), cudaMemcpyDeviceToHost, s));
    LORPC_CUDA(cudaStreamSynchronize(s));
    std::vector<int> rank((size_t)NT, -1);
    for (int i = 0; i < nint; ++i) rank[ilist[i]] = i;
    std::vector<double> F((size_t)nint * nint, 0.0);
    for (int i = 0; i < nint; ++i) {
      const long long g = ilist[i];
      for (int dd = 0; dd < ND; ++dd) {
        const long long h = g + dir_dx(dd) + (long long)nvl.x * (dir_dy(dd) + (long long)nvl.y * (d == 3 ? dir_dz(dd) : 0));
        if (h < 0 || h >= NT || rank[h] < 0) continue;
        F[(size_t)i * nint + rank[h]] = A[(size_t)g * ndp + dd];
      }
    }
    // Cholesky F = C C^T (lower, in place)
    for (int j = 0; j < nint; ++j) {
      double sj = F[(size_t)j * nint + j];
      for (int k = 0; k < j; ++k) sj -= F[(size_t)j * nint + k] * F[(size_t)j * nint + k];
      if (!(sj > 0.0)) return fail(LORPC_ERR_NOT_SPD, "coarsest GMG level: matrix not positive definite");
      const double cj = std::sqrt(sj);
      F[(size_t)j * nint + j] = cj;
      for (int i = j + 1; i < nint; ++i) {
        double t = F[(size_t)i * nint + j];
        for (int k = 0; k < j; ++k) t -= F[(size_t)i * nint + k] * F[(size_t)j * nint + k];
        F[(size_t)i * nint + j] = t / cj;
      }
    }
    // W = C^{-1} (lower), then inv = W^T W
    std::vector<double> W((size_t)nint * nint, 0.0);
    for (int j = 0; j < nint; ++j) {
      W[(size_t)j * nint + j] = 1.0 / F[(size_t)j * nint + j];
      for (int i = j + 1; i < nint; ++i) {
        double t = 0.0;
        for (int k = j; k < i; ++k) t += F[(size_t)i * nint + k] * W[(size_t)k * nint + j];
        W[(size_t)i * nint + j] = -t / F[(size_t)i * nint + i];
      }
    }
    std::vector<double> Inv((size_t)nint * nint, 0.0);
    for (int i = 0; i < nint; ++i)
      for (int j = 0; j <= i; ++j) {
        double t = 0.0;
        for (int k = i; k < nint; ++k) t += W[(size_t)k * nint + i] * W[(size_t)k * nint + j];
        Inv[(size_t)i * nint + j] = t;
        Inv[(size_t)j * nint + i] = t;
      }
    LORPC_CUDA(cudaMemcpyAsync(b->coarse_chol, Inv.data(), sizeof(double) * Inv.size(), cudaMemcpyHostToDevice, s));
    LORPC_CUDA(cudaMemcpyAsync(b->coarse_idx, ilist.data(), sizeof(int) * ilist.size(), cudaMemcpyHostToDevice, s));
    LORPC_CUDA(cudaStreamSynchronize(s));
  }
  return LORPC_OK;
}

int schwarz_build(lorpc_prec* b, cudaStream_t s) {
  const lorpc_mesh* m = b->m;
  const lorpc_lor* lor = b->lor;
  const int d = m->d, L = lor->L, ND = d == 2 ? 9 : 27;
  b->L = L;
  PatchGeom G = make_geom(b);
  if (b->desc.patch_kind == 0) {
    const int nvz = d == 3 ? m->n[2] + 1 : 1;
    if (b->pnvz <= 0) { b->pvz0 = 0; b->pnvz = nvz; }
    if (b->pvz0 < 0 || b->pvz0 + b->pnvz > nvz) return fail(LORPC_ERR_ARG, "schwarz: patch plane range");
    b->J = (long long)(m->n[0] + 1) * (m->n[1] + 1) * b->pnvz;
  } else if (b->desc.patch_kind == 2) {
    if (b->desc.coarse != 0) return fail(LORPC_ERR_ARG, "schwarz: B(1) needs R_0 (coarse = 0) at its bottom");
    b->pvz0 = 0; b->pnvz = 0;
    b->J = 1;
  } else {
    b->pvz0 = 0; b->pnvz = 0;
    b->J = m->nel;
  }
  // extended vertex patches (sec:aniso P:1123-1128, reading r6): along each axis, a
  // side of the patch shorter than half of the largest of its own elements on the
  // vertex line through x_j grows by one element layer at a time, <= 4 elements
  b->emax = b->desc.patch_kind == 0 ? 2 : 3;
  if (b->desc.extend) {
    if (b->desc.patch_kind != 0) return fail(LORPC_ERR_ARG, "schwarz: patch extension needs vertex patches");
    if (b->pnvz != (d == 3 ? m->n[2] + 1 : 1) || b->pvz0 != 0)
      return fail(LORPC_ERR_ARG, "schwarz: patch extension is single-rank only");
    const int nv[3] = {m->n[0] + 1, m->n[1] + 1, d == 3 ? m->n[2] + 1 : 1};
    std::vector<double> V((size_t)nv[0] * nv[1] * nv[2] * d);
    LORPC_CUDA(cudaMemcpy(V.data(), m->V, sizeof(double) * V.size(), cudaMemcpyDeviceToHost));
    b->erng_h.assign((size_t)b->J * 6, 0);
    b->emax = 1;
    for (long long j = 0; j < b->J; ++j) {
      const int vc[3] = {(int)(j % nv[0]), (int)((j / nv[0]) % nv[1]), (int)(j / ((long long)nv[0] * nv[1]))};
      for (int k = 0; k < d; ++k) {
        auto xk = [&](int i) {
          int g[3] = {vc[0], vc[1], vc[2]};
          g[k] = i;
          return V[((size_t)g[0] + (size_t)nv[0] * (g[1] + (size_t)nv[1] * g[2])) * d + k];
        };
        int lo = std::max(vc[k] - 1, 0), hi = std::min(vc[k], m->n[k] - 1);
        double H = 0.0;
        for (int i = lo; i <= hi; ++i) H = std::max(H, xk(i + 1) - xk(i));
        if (vc[k] > 0)
          while (xk(vc[k]) - xk(lo) < 0.5 * H && lo > 0 && hi - lo + 1 < 4) --lo;
        if (vc[k] < m->n[k])
          while (xk(hi + 1) - xk(vc[k]) < 0.5 * H && hi < m->n[k] - 1 && hi - lo + 1 < 4) ++hi;
        b->erng_h[6 * j + 2 * k] = (short)lo;
        b->erng_h[6 * j + 2 * k + 1] = (short)hi;
        b->emax = std::max(b->emax, hi - lo + 1);
      }
    }
    LORPC_TRY(dalloc(&b->erng, b->erng_h.size()));
    LORPC_CUDA(cudaMemcpy(b->erng, b->erng_h.data(), sizeof(short) * b->erng_h.size(), cudaMemcpyHostToDevice));
    G.erng = b->erng;
  }
  PatchGeom Gh = G;  // host copy of the geometry for the record sizes
  if (b->desc.extend) Gh.erng = b->erng_h.data();
  // record offsets (host; patch sizes are index arithmetic)
  b->recoff_h.assign((size_t)b->J * L, 0);
  long long off = 0;
  for (int l = 0; l < MAXL; ++l) b->max_n[l] = 0;
  b->rec_max = 0;
  for (long long j = 0; j < b->J; ++j) {
    const long long start = off;
    for (int l = 0; l < L; ++l) {
      int lo[3], ext[3];
      patch_box(Gh, j, l, lo, ext);
      const int n = std::max(ext[0] * ext[1] * ext[2], 0);
      if (n > 65535) return fail(LORPC_ERR_SIZE, "patch too large");
      if (num_edges(d, ext) > 65535)  // record row offsets (frp / brp) are u16
        return fail(LORPC_ERR_SIZE, "patch has more than 65535 stencil edges");
      b->max_n[l] = std::max(b->max_n[l], n);
      b->recoff_h[j * L + l] = off;
      const long long nL = num_edges(d, ext);
      b->factor_values += n + nL;
      off += rec_layout(n, nL).total;
    }
    b->rec_max = std::max(b->rec_max, off - start);
  }
  b->rec_bytes = off;
  LORPC_TRY(dalloc(&b->rec, (size_t)off));
  LORPC_TRY(dalloc(&b->recoff, b->recoff_h.size()));
  LORPC_CUDA(cudaMemcpyAsync(b->recoff, b->recoff_h.data(), sizeof(long long) * b->recoff_h.size(),
                             cudaMemcpyHostToDevice, s));
  // MDF + ILU(0) batch
  int maxn = 1;
  for (int l = 0; l < L; ++l) maxn = std::max(maxn, b->max_n[l]);
  int dev, nsm;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  long long ntasks = b->J * L;
  long long nwarps = std::min<long long>(ntasks, (long long)nsm * 16);
  // cap scratch at ~2 GB
  const long long per_warp = (long long)maxn * (2 * ND + 1) * 8 + ((5ll + ND) * maxn + 1) * 4 + maxn;
  nwarps = std::max<long long>(1, std::min<long long>(nwarps, (2ll << 30) / per_warp));
  MdfParams P{};
  P.G = G;
  for (int l = 0; l < L; ++l) P.A[l] = lor->A[l];
  P.rec = b->rec; P.recoff = b->recoff; P.ntasks = ntasks; P.ordering = b->desc.ordering; P.maxn = maxn;
  LORPC_TRY(dalloc(&P.scratch, (size_t)nwarps * maxn * (2 * ND + 1)));
  LORPC_TRY(dalloc(&P.iscratch, (size_t)nwarps * ((5 + ND) * maxn + 1)));
  LORPC_TRY(dalloc(&P.alive, (size_t)nwarps * maxn));
  LORPC_TRY(dalloc(&P.err, 1));
  LORPC_TRY(dalloc(&P.err_step, 1));
  LORPC_CUDA(cudaMemsetAsync(P.err, 0xff, sizeof(unsigned long long), s));
  const unsigned blocks = (unsigned)((nwarps * 32 + 127) / 128);
  if (d == 2) k_mdf_ilu<2><<<blocks, 128, 0, s>>>(P); else k_mdf_ilu<3><<<blocks, 128, 0, s>>>(P);
  LORPC_LAUNCHED();
  unsigned long long err = 0;
  int estep = 0;
  LORPC_CUDA(cudaMemcpyAsync(&err, P.err, sizeof(err), cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaMemcpyAsync(&estep, P.err_step, sizeof(int), cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  dfree(P.scratch); dfree(P.iscratch); dfree(P.alive); dfree(P.err); dfree(P.err_step);
  if (err != ~0ull)
    return fail(LORPC_ERR_ZERO_PIVOT, "ilu: non-positive pivot (patch " + std::to_string(err / L) + ", level " +
                                          std::to_string(err % L) + ", step " + std::to_string(estep) + ")");
  // separable patch transfer tables.  A patch box starts at an element boundary,
  // so its 1D restriction depends only on the level and on the number e of
  // elements along the axis: W[ic][f] = P_l(f, ic) on the free nodes of e elements.
  {
    std::vector<double> W;
    const int emax = b->emax;
    b->scratch_doubles = 0;
    for (int l = 0; l + 1 < L; ++l) {
      const Transfer1D& T = lor->T[l];
      const int mf = lor->ml[l], mc = lor->ml[l + 1];
      for (int e = 0; e < 5; ++e) { b->woff[l][e] = 0; b->wfe[l][e] = 0; b->wce[l][e] = 0; }
      for (int e = 1; e <= 4; ++e) {
        const int fe = e * (mf - 1) - 1, ce = e * (mc - 1) - 1;
        b->woff[l][e] = (int)W.size(); b->wfe[l][e] = fe; b->wce[l][e] = ce;
        W.resize(W.size() + (size_t)std::max(fe * ce, 0), 0.0);
        double* w = W.data() + b->woff[l][e];
        for (int f = 0; f < fe; ++f) {
          const int gf = f + 1;
          const int el = std::min(gf / (mf - 1), e - 1);
          const int t = gf - el * (mf - 1);
          const int c0 = el * (mc - 1) + T.c0[t] - 1, c1 = el * (mc - 1) + T.c1[t] - 1;
          if (c0 >= 0 && c0 < ce) w[c0 * fe + f] += T.w0[t];
          if (c1 != c0 && c1 >= 0 && c1 < ce) w[c1 * fe + f] += T.w1[t];
        }
      }
      const int fe = emax * (mf - 1) - 1, ce = emax * (mc - 1) - 1;
      const int sc = d == 3 ? ce * fe * fe + ce * ce * fe : ce * fe;
      b->scratch_doubles = std::max(b->scratch_doubles, sc);
    }
    if (W.empty()) W.push_back(0.0);
    LORPC_TRY(dalloc(&b->wtab, W.size()));
    LORPC_CUDA(cudaMemcpyAsync(b->wtab, W.data(), sizeof(double) * W.size(), cudaMemcpyHostToDevice, s));
    LORPC_CUDA(cudaStreamSynchronize(s));
    // lanes per patch: ~ the mean DAG-level width of the finest records is 3-6
    // rows; larger patches get more lanes so the shared footprint per warp stays small
    int per_patch = b->scratch_doubles;
    for (int l = 0; l < L; ++l) per_patch += 3 * b->max_n[l];
    (void)per_patch;
    // measured best among {4, 8, 16, 32} lanes (r01 probe): C5 (125-node patches) 16, C3 (343) 32
    b->lanes = 32;  // with 64-register V-cycle kernels (r01 probe: C5 161 ms vs 202 ms at G=16)
    if (const char* e = getenv("LORPC_LANES")) b->lanes = atoi(e);
  }
  // coarse space hierarchy (reading c11): level 0 = last LOR level (vertex grid)
  b->nc = 0;
  for (int i = 0; i < MAXC; ++i) { b->Ac[i] = b->dl1[i] = b->cr[i] = b->cz[i] = b->cs[i] = nullptr; }
  if (b->desc.coarse == 0) {
    const int nv[3] = {m->n[0] + 1, m->n[1] + 1, d == 3 ? m->n[2] + 1 : 1};
    LORPC_TRY(gmg_build(b, lor->A[L - 1], nv, d, s));
  }
  if (b->desc.patch_kind == 2) return single_setup(b);  // B(1): level-grid V-cycle (single.cu)
  // dense coarse V-cycle operators: first level l >= 1 with <= 32 free nodes per patch
  // (the coarsest level if none); the V-cycle below it is one symmetric matrix
  b->Ld = L - 1;
  for (int l = 1; l < L; ++l)
    if (b->max_n[l] <= 32) { b->Ld = l; break; }
  if (b->max_n[b->Ld] > 64) return fail(LORPC_ERR_SIZE, "dense coarse level too large");
  b->ldc = std::max(b->max_n[b->Ld] * b->max_n[b->Ld], 1);
  LORPC_TRY(dalloc(&b->Cd, (size_t)b->J * b->ldc));
  LORPC_TRY(dense_coarse_setup(b, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  // warp-per-patch fused V-cycle (vcycle_w.cu): 3D vertex patches with a level-1 box
  // of at most 3 x 3 x 3 nodes (p = 3) and node indices that fit in a byte
  {
    const int cx = 2 * (lor->ml[1] - 1) - 1;
    // opt-in (LORPC_WMODE=1): parity-exact, but measured slower than the thread-mode
    // kernels on C5: only ~14 patches fit per SM with their factor
    // resident, and the push-round chains are latency-bound
    const bool eligible = d == 3 && b->desc.patch_kind == 0 && !b->desc.extend && b->Ld == 1 && cx <= 3 &&
                          b->max_n[0] <= 255;
    const char* e = getenv("LORPC_WMODE");
    b->wmode = eligible && e && atoi(e) != 0;
    if (b->wmode) {
      LORPC_TRY(wrec_build(b, s));
      if (wmode_smem(b) > 227 * 1024) return fail(LORPC_ERR_SIZE, "wmode: record does not fit in shared memory");
      return LORPC_OK;
    }
    // Q mode (LP lanes per patch, factors streamed through a cp.async ring): structure-only
    // orderings (natural, RCM) on the same patches; LORPC_QMODE=0 disables it
    const char* eq = getenv("LORPC_QMODE");
    if (eligible && b->desc.ordering != 0 && eq && atoi(eq) != 0) {
      int ok = 0;
      LORPC_TRY(qrec_build(b, s, &ok));
      if (ok && qmode_smem(b) <= 227 * 1024) {
        b->qmode = true;
        return LORPC_OK;
      }
      if (ok) return fail(LORPC_ERR_SIZE, "qmode: shared memory");
    }
  }
  // thread-per-patch V-cycle when the warp's 32 patch vectors fit in shared memory
  // (level-1 boxes of at most 3 (3D) / 5 (2D) nodes per axis, see vcycle_t.cu TCoarse)
  const int cext_max = b->emax * (lor->ml[1] - 1) - 1;
  b->tmode = b->Ld == 1 && b->max_n[1] <= 32 && cext_max <= (d == 3 ? 3 : 5) && tmode_smem(b) <= 227 * 1024 &&
             b->max_n[0] <= 65534;
  if (const char* e = getenv("LORPC_TMODE")) b->tmode = b->tmode && atoi(e) != 0;
  if (b->tmode) LORPC_TRY(trec_build(b, s));
  return LORPC_OK;
}


int export_ordering(const lorpc_prec* b, long long j, int l, int* perm, int* n) {
  if (j < 0 || j >= b->J || l < 0 || l >= b->L) return fail(LORPC_ERR_ARG, "export_ordering: bad patch/level");
  const long long off = b->recoff_h[j * b->L + l];
  int h[4];
  LORPC_CUDA(cudaMemcpy(h, b->rec + off, sizeof(h), cudaMemcpyDeviceToHost));
  if (*n < h[0]) { *n = h[0]; return fail(LORPC_ERR_ARG, "export_ordering: buffer too small"); }
  *n = h[0];
  if (h[0] == 0) return LORPC_OK;
  const RecLayout R = rec_layout(h[0], h[2]);
  std::vector<uint16_t> o(h[0]);
  LORPC_CUDA(cudaMemcpy(o.data(), b->rec + off + R.order, 2 * h[0], cudaMemcpyDeviceToHost));
  for (int i = 0; i < h[0]; ++i) perm[i] = o[i];
  return LORPC_OK;
}

}  // namespace lorpc

