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
#include <cstring>

#include "device.cuh"

namespace lorpc {

int galerkin(int d, const double* Af, double* Ac, const Transfer1D& T, const int* ne, const int* Nf, const int* Nc,
             cudaStream_t s);
Transfer1D gmg_transfer();

// ------------------------------------------------------------------ patch geometry
struct PatchGeom {
  int d, kind;          // kind 0 vertex, 1 star
  int n[3];             // elements per axis
  int ml[MAXL];         // nodes per element per axis at each level
  int Nax[MAXL][3];     // level grid per axis
  int L;
};

__host__ __device__ __forceinline__ void patch_elems(const PatchGeom& G, long long j, int* elo, int* ehi) {
  if (G.kind == 0) {
    const long long nv0 = G.n[0] + 1, nv1 = G.n[1] + 1;
    const int v[3] = {(int)(j % nv0), (int)((j / nv0) % nv1), (int)(j / (nv0 * nv1))};
    for (int k = 0; k < 3; ++k) {
      if (k >= G.d) { elo[k] = ehi[k] = 0; continue; }
      elo[k] = v[k] - 1 < 0 ? 0 : v[k] - 1;
      ehi[k] = v[k] < G.n[k] - 1 ? v[k] : G.n[k] - 1;
    }
  } else {
    const int e[3] = {(int)(j % G.n[0]), (int)((j / G.n[0]) % G.n[1]), (int)(j / ((long long)G.n[0] * G.n[1]))};
    for (int k = 0; k < 3; ++k) {
      if (k >= G.d) { elo[k] = ehi[k] = 0; continue; }
      elo[k] = e[k] - 1 < 0 ? 0 : e[k] - 1;
      ehi[k] = e[k] + 1 < G.n[k] - 1 ? e[k] + 1 : G.n[k] - 1;
    }
  }
}
// free node box at level l: first free node lo[k] (level-global), extent ext[k]
__host__ __device__ __forceinline__ void patch_box(const PatchGeom& G, long long j, int l, int* lo, int* ext) {
  int elo[3], ehi[3];
  patch_elems(G, j, elo, ehi);
  const int m = G.ml[l];
  for (int k = 0; k < 3; ++k) {
    if (k >= G.d) { lo[k] = 0; ext[k] = 1; continue; }
    lo[k] = elo[k] * (m - 1) + 1;
    ext[k] = (ehi[k] - elo[k] + 1) * (m - 1) - 1;
  }
}
__host__ __device__ __forceinline__ long long num_edges(int d, const int* ext) {
  // half-stencil directions: lexicographically positive offsets
  long long s = 0;
  for (int dz = (d == 3 ? -1 : 0); dz <= (d == 3 ? 1 : 0); ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const bool pos = dz > 0 || (dz == 0 && (dy > 0 || (dy == 0 && dx > 0)));
        if (!pos) continue;
        long long c = 1;
        const int o[3] = {dx, dy, dz};
        for (int k = 0; k < d; ++k) { int v = ext[k] - (o[k] < 0 ? -o[k] : o[k]); c *= v > 0 ? v : 0; }
        s += c;
      }
  return s;
}
__host__ __device__ __forceinline__ long long a8(long long b) { return (b + 7) & ~7ll; }
struct RecLayout { long long D, L, mask, off, sched, lptr, order, total; };
__host__ __device__ __forceinline__ RecLayout rec_layout(int n, long long nL) {
  RecLayout R;
  R.D = 16;
  R.L = R.D + 8ll * n;
  R.mask = R.L + 8ll * nL;
  R.off = R.mask + a8(4ll * n);
  R.sched = R.off + a8(2ll * n);
  R.lptr = R.sched + a8(2ll * n);
  R.order = R.lptr + a8(2ll * (n + 1));
  R.total = R.order + a8(2ll * n);
  return R;
}

// ------------------------------------------------------------------ MDF + ILU(0)
__device__ __forceinline__ double q30(double x) {
  if (x == 0.0) return 0.0;
  int e;
  const double f = frexp(x, &e);
  return ldexp(rint(ldexp(f, 30)), e - 30);
}

template <int DIM>
__device__ __forceinline__ int doff(int d, int ex, int ey) {
  return dir_dx(d) + ex * (dir_dy(d) + ey * (DIM == 3 ? dir_dz(d) : 0));
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
  int* iscratch;        // per warp: pos[maxn], lev[maxn], order[maxn], cnt[maxn+1]
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
  int* pos = P.iscratch + gw * (long long)(4 * P.maxn + 1);
  int* lev = pos + P.maxn;
  int* ord = lev + P.maxn;
  int* cnt = ord + P.maxn;
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
    const long long NT = Nx * Ny * P.G.Nax[l][2];
    const double* A = P.A[l];
    for (int i = lane; i < n; i += 32) {
      const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
      const long long gi = (lo[0] + ix) + Nx * ((lo[1] + iy) + Ny * (DIM == 3 ? lo[2] + iz : 0));
      const uint32_t em = exist_mask<DIM>(ix, iy, iz, ex, ey, ez);
      for (int d = 0; d < ND; ++d) {
        At[i * ND + d] = ((em >> d) & 1u) ? A[(long long)d * NT + gi] : 0.0;
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
    __syncwarp();
    bool failed = false;
    for (int step = 0; step < n; ++step) {
      double bk = INFINITY;
      int bi = 0x7fffffff;
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
    // ---- record: pivots D (natural order) stored from the final At diagonal
    double* Dr = (double*)(rec + R.D);
    double* Lr = (double*)(rec + R.L);
    uint32_t* mr = (uint32_t*)(rec + R.mask);
    uint16_t* offr = (uint16_t*)(rec + R.off);
    uint16_t* sch = (uint16_t*)(rec + R.sched);
    uint16_t* lpt = (uint16_t*)(rec + R.lptr);
    uint16_t* orr = (uint16_t*)(rec + R.order);
    for (int i = lane; i < n; i += 32) {
      Dr[i] = At[i * ND + C];  // pivot at elimination time (never modified afterwards)
      orr[i] = (uint16_t)ord[i];
    }
    if (lane == 0) {
      // lower masks, compact L values, offsets, DAG levels (in step order)
      int depth = 0;
      for (int i = 0; i < n; ++i) cnt[i] = 0;
      int off = 0;
      for (int i = 0; i < n; ++i) {
        const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
        const uint32_t em = exist_mask<DIM>(ix, iy, iz, ex, ey, ez);
        uint32_t lm = 0;
        for (int d = 0; d < ND; ++d) {
          if (d == C || !((em >> d) & 1u)) continue;
          const int jn = i + doff<DIM>(d, ex, ey);
          if (pos[jn] < pos[i]) { lm |= 1u << d; Lr[off++] = Lf[i * ND + d]; }
        }
        mr[i] = lm;
        offr[i] = (uint16_t)(off - __popc(lm));
      }
      for (int t = 0; t < n; ++t) {
        const int i = ord[t];
        const int ix = i % ex, iy = (i / ex) % ey;
        int lv = 0;
        uint32_t lm = mr[i];
        while (lm) {
          const int d = __ffs(lm) - 1;
          lm &= lm - 1;
          const int jn = i + doff<DIM>(d, ex, ey);
          lv = max(lv, lev[jn] + 1);
        }
        (void)ix; (void)iy;
        lev[i] = lv;
        depth = max(depth, lv + 1);
        cnt[lv]++;
      }
      // level pointers + stable placement in step order
      int acc = 0;
      for (int v = 0; v < depth; ++v) { lpt[v] = (uint16_t)acc; const int c = cnt[v]; cnt[v] = acc; acc += c; }
      lpt[depth] = (uint16_t)acc;
      for (int t = 0; t < n; ++t) { const int i = ord[t]; sch[cnt[lev[i]]++] = (uint16_t)i; }
      int* h = (int*)rec;
      h[0] = n; h[1] = depth; h[2] = (int)nL; h[3] = l;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ V-cycle apply
struct VcParams {
  PatchGeom G;
  const double* A[MAXL];
  Transfer1D T[MAXL];
  const char* rec;
  const long long* recoff;
  long long J;
  int soff[MAXL];       // shared-memory offsets (doubles) of level vectors per warp
  int warp_doubles;
  const double* r;
  double* z;
};

template <int DIM>
__device__ void ilu_solve(const char* rec, double* v, int ex, int ey, int ez, int lane) {
  constexpr int ND = Dirs<DIM>::ND, C = Dirs<DIM>::CENTER;
  const int* h = (const int*)rec;
  const int n = h[0], depth = h[1];
  if (n == 0) return;
  const RecLayout R = rec_layout(n, h[2]);
  const double* D = (const double*)(rec + R.D);
  const double* L = (const double*)(rec + R.L);
  const uint32_t* lm = (const uint32_t*)(rec + R.mask);
  const uint16_t* off = (const uint16_t*)(rec + R.off);
  const uint16_t* sch = (const uint16_t*)(rec + R.sched);
  const uint16_t* lpt = (const uint16_t*)(rec + R.lptr);
  // forward: L y = r
  for (int lv = 0; lv < depth; ++lv) {
    const int b = lpt[lv], e = lpt[lv + 1];
    for (int t = b + lane; t < e; t += 32) {
      const int i = sch[t];
      double acc = v[i];
      uint32_t m = lm[i];
      int o = off[i];
      while (m) {
        const int d = __ffs(m) - 1;
        m &= m - 1;
        acc -= L[o++] * v[i + doff<DIM>(d, ex, ey)];
      }
      v[i] = acc;
    }
    __syncwarp();
  }
  for (int i = lane; i < n; i += 32) v[i] = v[i] / D[i];
  __syncwarp();
  // backward: L^T z = y
  for (int lv = depth - 1; lv >= 0; --lv) {
    const int b = lpt[lv], e = lpt[lv + 1];
    for (int t = b + lane; t < e; t += 32) {
      const int i = sch[t];
      const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
      uint32_t um = exist_mask<DIM>(ix, iy, iz, ex, ey, ez) & ~lm[i] & ~(1u << C);
      double acc = v[i];
      while (um) {
        const int d = __ffs(um) - 1;
        um &= um - 1;
        const int k = i + doff<DIM>(d, ex, ey);
        const int rev = ND - 1 - d;
        const double lki = L[off[k] + __popc(lm[k] & ((1u << rev) - 1u))];
        acc -= lki * v[k];
      }
      v[i] = acc;
    }
    __syncwarp();
  }
}

template <int DIM>
__device__ void residual(const double* A, long long Nx, long long Ny, long long NT, const int* lo, const int* ext,
                         const double* r, const double* z, double* s, int lane) {
  constexpr int ND = Dirs<DIM>::ND;
  const int ex = ext[0], ey = ext[1], ez = ext[2], n = ex * ey * ez;
  for (int i = lane; i < n; i += 32) {
    const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
    const long long gi = (lo[0] + ix) + Nx * ((lo[1] + iy) + Ny * (DIM == 3 ? lo[2] + iz : 0));
    uint32_t em = exist_mask<DIM>(ix, iy, iz, ex, ey, ez);
    double acc = r[i];
    while (em) {
      const int d = __ffs(em) - 1;
      em &= em - 1;
      acc -= A[(long long)d * NT + gi] * z[i + doff<DIM>(d, ex, ey)];
    }
    s[i] = acc;
  }
}

__device__ __forceinline__ void targets1(const Transfer1D& T, int ne, int f, int& c0, int& c1, double& w0, double& w1) {
  const int e = min(f / (T.mf - 1), ne - 1);
  const int t = f - e * (T.mf - 1);
  const int base = e * (T.mc - 1);
  c0 = base + T.c0[t]; c1 = base + T.c1[t]; w0 = T.w0[t]; w1 = T.w1[t];
}
__device__ __forceinline__ double weight1(const Transfer1D& T, int ne, int f, int ic) {
  int c0, c1; double w0, w1;
  targets1(T, ne, f, c0, c1, w0, w1);
  double w = 0.0;
  if (c0 == ic) w += w0;
  if (c1 == ic && c1 != c0) w += w1;
  return w;
}
__device__ __forceinline__ int fpos1(const Transfer1D& T, int ne, int ic) {
  const int e = min(ic / (T.mc - 1), ne - 1);
  return e * (T.mf - 1) + T.ret[ic - e * (T.mc - 1)];
}

template <int DIM>
__global__ void __launch_bounds__(128) k_vcycle(VcParams P) {
  constexpr int ND = Dirs<DIM>::ND;
  (void)ND;
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long j = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (j >= P.J) return;
  double* W = sm + (long long)wib * P.warp_doubles;
  const int L = P.G.L;
  int lo[MAXL][3], ext[MAXL][3], nn[MAXL];
  for (int l = 0; l < L; ++l) {
    patch_box(P.G, j, l, lo[l], ext[l]);
    nn[l] = ext[l][0] * ext[l][1] * ext[l][2];
    if (nn[l] < 0) nn[l] = 0;
  }
  auto rv = [&](int l) { return W + P.soff[l]; };
  auto zv = [&](int l) { return W + P.soff[l] + nn[l]; };
  auto sv = [&](int l) { return W + P.soff[l] + 2 * nn[l]; };
  // gather r_j = I_j^T r (a5)
  {
    const long long Nx = P.G.Nax[0][0], Ny = P.G.Nax[0][1];
    const int ex = ext[0][0], ey = ext[0][1];
    double* r0 = rv(0);
    for (int i = lane; i < nn[0]; i += 32) {
      const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
      const long long gi = (lo[0][0] + ix) + Nx * ((lo[0][1] + iy) + Ny * (DIM == 3 ? lo[0][2] + iz : 0));
      r0[i] = P.r[gi];
    }
  }
  __syncwarp();
  // downward leg
  for (int l = 0; l < L - 1; ++l) {
    const char* rec = P.rec + P.recoff[j * L + l];
    double *r = rv(l), *z = zv(l), *s = sv(l);
    const int ex = ext[l][0], ey = ext[l][1], ez = ext[l][2];
    for (int i = lane; i < nn[l]; i += 32) z[i] = r[i];
    __syncwarp();
    ilu_solve<DIM>(rec, z, ex, ey, ez, lane);                        // pre-smoothing
    const long long Nx = P.G.Nax[l][0], Ny = P.G.Nax[l][1], NT = Nx * Ny * P.G.Nax[l][2];
    residual<DIM>(P.A[l], Nx, Ny, NT, lo[l], ext[l], r, z, s, lane);
    __syncwarp();
    // restriction r_{l+1} = P^T s
    const Transfer1D& T = P.T[l];
    double* rc = rv(l + 1);
    const int cx = ext[l + 1][0], cy = ext[l + 1][1];
    for (int I = lane; I < nn[l + 1]; I += 32) {
      const int Ic[3] = {lo[l + 1][0] + I % cx, lo[l + 1][1] + (I / cx) % cy, lo[l + 1][2] + I / (cx * cy)};
      int flo[3] = {0, 0, 0}, fhi[3] = {0, 0, 0};
      for (int k = 0; k < DIM; ++k) {
        const int fp = fpos1(T, P.G.n[k], Ic[k]);
        flo[k] = max(fp - T.gap, lo[l][k]);
        fhi[k] = min(fp + T.gap, lo[l][k] + ext[l][k] - 1);
      }
      double acc = 0.0;
      for (int fz = flo[2]; fz <= fhi[2]; ++fz) {
        const double wz = DIM == 3 ? weight1(T, P.G.n[2], fz, Ic[2]) : 1.0;
        if (wz == 0.0) continue;
        for (int fy = flo[1]; fy <= fhi[1]; ++fy) {
          const double wy = weight1(T, P.G.n[1], fy, Ic[1]);
          if (wy == 0.0) continue;
          for (int fx = flo[0]; fx <= fhi[0]; ++fx) {
            const double wx = weight1(T, P.G.n[0], fx, Ic[0]);
            if (wx == 0.0) continue;
            const int li = (fx - lo[l][0]) + ex * ((fy - lo[l][1]) + ey * (DIM == 3 ? fz - lo[l][2] : 0));
            acc += wx * wy * wz * s[li];
          }
        }
      }
      rc[I] = acc;
    }
    __syncwarp();
  }
  // coarsest level: exact LDL^T (reading c8)
  {
    const int l = L - 1;
    double *r = rv(l), *z = zv(l);
    for (int i = lane; i < nn[l]; i += 32) z[i] = r[i];
    __syncwarp();
    ilu_solve<DIM>(P.rec + P.recoff[j * L + l], z, ext[l][0], ext[l][1], ext[l][2], lane);
  }
  // upward leg
  for (int l = L - 2; l >= 0; --l) {
    const char* rec = P.rec + P.recoff[j * L + l];
    double *r = rv(l), *z = zv(l), *s = sv(l);
    const double* zc = zv(l + 1);
    const Transfer1D& T = P.T[l];
    const int ex = ext[l][0], ey = ext[l][1], ez = ext[l][2];
    const int cx = ext[l + 1][0], cy = ext[l + 1][1], cz = ext[l + 1][2];
    for (int i = lane; i < nn[l]; i += 32) {                          // z += P z_{l+1}
      const int f[3] = {lo[l][0] + i % ex, lo[l][1] + (i / ex) % ey, lo[l][2] + i / (ex * ey)};
      int c0[3] = {0, 0, 0}, c1[3] = {0, 0, 0};
      double w0[3] = {1, 1, 1}, w1[3] = {0, 0, 0};
      for (int k = 0; k < DIM; ++k) targets1(T, P.G.n[k], f[k], c0[k], c1[k], w0[k], w1[k]);
      double acc = 0.0;
      for (int sel = 0; sel < (1 << DIM); ++sel) {
        double w = 1.0;
        int cl[3] = {0, 0, 0};
        bool ok = true;
        for (int k = 0; k < DIM; ++k) {
          const int b = (sel >> k) & 1;
          if (b && c1[k] == c0[k]) { ok = false; break; }
          const int c = (b ? c1[k] : c0[k]) - lo[l + 1][k];
          const int ce = k == 0 ? cx : (k == 1 ? cy : cz);
          if (c < 0 || c >= ce) { ok = false; break; }
          w *= b ? w1[k] : w0[k];
          cl[k] = c;
        }
        if (!ok) continue;
        acc += w * zc[cl[0] + cx * (cl[1] + cy * cl[2])];
      }
      z[i] += acc;
    }
    __syncwarp();
    const long long Nx = P.G.Nax[l][0], Ny = P.G.Nax[l][1], NT = Nx * Ny * P.G.Nax[l][2];
    residual<DIM>(P.A[l], Nx, Ny, NT, lo[l], ext[l], r, z, s, lane);
    __syncwarp();
    ilu_solve<DIM>(rec, s, ex, ey, ez, lane);                         // post-smoothing
    for (int i = lane; i < nn[l]; i += 32) z[i] += s[i];
    __syncwarp();
  }
  // z += I_j z_j (a8)
  {
    const long long Nx = P.G.Nax[0][0], Ny = P.G.Nax[0][1];
    const int ex = ext[0][0], ey = ext[0][1];
    const double* z0 = zv(0);
    for (int i = lane; i < nn[0]; i += 32) {
      const int ix = i % ex, iy = (i / ex) % ey, iz = i / (ex * ey);
      const long long gi = (lo[0][0] + ix) + Nx * ((lo[0][1] + iy) + Ny * (DIM == 3 ? lo[0][2] + iz : 0));
      atomicAdd(P.z + gi, z0[i]);
    }
  }
}

// ------------------------------------------------------------------ coarse space R_0
// P_0^T r: vertex v gathers the LOR nodes of its 2^d adjacent elements with the
// multilinear hat weights in the GLL reference coordinate.
template <int DIM>
__global__ void k_restrict_vertex(const double* __restrict__ r, double* __restrict__ rc, int3 nv, int3 N, Basis1D bs) {
  const long long NV = (long long)nv.x * nv.y * nv.z;
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= NV) return;
  const int vc[3] = {(int)(v % nv.x), (int)((v / nv.x) % nv.y), (int)(v / ((long long)nv.x * nv.y))};
  const int Nn[3] = {N.x, N.y, N.z}, nvv[3] = {nv.x, nv.y, nv.z};
  bool interior = true;
  for (int k = 0; k < DIM; ++k) if (vc[k] == 0 || vc[k] == nvv[k] - 1) interior = false;
  if (!interior) { rc[v] = 0.0; return; }
  const int p = bs.p;
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int k = 0; k < DIM; ++k) { lo[k] = (vc[k] - 1) * p + 1; hi[k] = (vc[k] + 1) * p - 1; }
  double acc = 0.0;
  for (int gz = lo[2]; gz <= hi[2]; ++gz) {
    double wz = 1.0;
    if (DIM == 3) { const int t = gz - vc[2] * p; wz = t <= 0 ? bs.xi[t + p] : 1.0 - bs.xi[t]; }
    for (int gy = lo[1]; gy <= hi[1]; ++gy) {
      const int ty = gy - vc[1] * p;
      const double wy = ty <= 0 ? bs.xi[ty + p] : 1.0 - bs.xi[ty];
      for (int gx = lo[0]; gx <= hi[0]; ++gx) {
        const int tx = gx - vc[0] * p;
        const double wx = tx <= 0 ? bs.xi[tx + p] : 1.0 - bs.xi[tx];
        acc += wx * wy * wz * r[gx + (long long)Nn[0] * (gy + (long long)Nn[1] * gz)];
      }
    }
  }
  rc[v] = acc;
}

// z += P_0 z_0, then z_D = 0
template <int DIM>
__global__ void k_prolong_vertex_add(const double* __restrict__ zc, double* __restrict__ z, int3 nv, int3 N, int3 n,
                                     Basis1D bs) {
  const long long NT = (long long)N.x * N.y * N.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NT) return;
  const int gc[3] = {(int)(g % N.x), (int)((g / N.x) % N.y), (int)(g / ((long long)N.x * N.y))};
  const int Nn[3] = {N.x, N.y, N.z}, nn[3] = {n.x, n.y, n.z};
  bool dir = false;
  for (int k = 0; k < DIM; ++k) if (gc[k] == 0 || gc[k] == Nn[k] - 1) dir = true;
  if (dir) { z[g] = 0.0; return; }
  const int p = bs.p;
  int v0[3] = {0, 0, 0};
  double w0[3] = {1, 1, 1}, w1[3] = {0, 0, 0};
  for (int k = 0; k < DIM; ++k) {
    const int e = min(gc[k] / p, nn[k] - 1);
    const int a = gc[k] - e * p;
    v0[k] = e; w0[k] = 1.0 - bs.xi[a]; w1[k] = bs.xi[a];
  }
  double acc = 0.0;
  for (int sel = 0; sel < (1 << DIM); ++sel) {
    double w = 1.0;
    int vv[3] = {0, 0, 0};
    for (int k = 0; k < DIM; ++k) {
      const int b = (sel >> k) & 1;
      w *= b ? w1[k] : w0[k];
      vv[k] = v0[k] + b;
    }
    if (w == 0.0) continue;
    acc += w * zc[vv[0] + (long long)nv.x * (vv[1] + (long long)nv.y * vv[2])];
  }
  z[g] += acc;
}

// l1-Jacobi diagonal over interior columns of interior rows
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
    if (in) s += fabs(A[(long long)d * NT + g]);
  }
  dl[g] = s;
}

// GMG smoothing kernels on a vertex grid (interior nodes; boundary nodes hold 0)
template <int DIM>
__device__ __forceinline__ bool interior_of(long long g, int3 Nv, int* c) {
  c[0] = (int)(g % Nv.x); c[1] = (int)((g / Nv.x) % Nv.y); c[2] = (int)(g / ((long long)Nv.x * Nv.y));
  bool in = c[0] > 0 && c[0] < Nv.x - 1 && c[1] > 0 && c[1] < Nv.y - 1;
  if (DIM == 3) in = in && c[2] > 0 && c[2] < Nv.z - 1;
  return in;
}
template <int DIM>
__device__ __forceinline__ double stencil_apply(const double* A, const double* z, long long g, int3 Nv, long long NT) {
  constexpr int ND = Dirs<DIM>::ND;
  double acc = 0.0;
  for (int d = 0; d < ND; ++d) {
    const long long o = dir_dx(d) + (long long)Nv.x * (dir_dy(d) + (long long)Nv.y * (DIM == 3 ? dir_dz(d) : 0));
    acc += A[(long long)d * NT + g] * z[g + o];
  }
  return acc;
}
// mode 0: z = r / d ; s = (later) ;  mode 1: s = r - A z ; mode 2: z += (r - A z)/d written to s then copied
template <int DIM>
__global__ void k_jacobi_pre(const double* __restrict__ r, const double* __restrict__ dl, double* __restrict__ z, int3 Nv) {
  const long long NT = (long long)Nv.x * Nv.y * Nv.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NT) return;
  int c[3];
  z[g] = interior_of<DIM>(g, Nv, c) ? r[g] / dl[g] : 0.0;
}
template <int DIM>
__global__ void k_residual_grid(const double* __restrict__ A, const double* __restrict__ r, const double* __restrict__ z,
                                double* __restrict__ s, int3 Nv) {
  const long long NT = (long long)Nv.x * Nv.y * Nv.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NT) return;
  int c[3];
  s[g] = interior_of<DIM>(g, Nv, c) ? r[g] - stencil_apply<DIM>(A, z, g, Nv, NT) : 0.0;
}
template <int DIM>
__global__ void k_jacobi_post(const double* __restrict__ A, const double* __restrict__ r, const double* __restrict__ dl,
                              const double* __restrict__ z, double* __restrict__ znew, int3 Nv) {
  const long long NT = (long long)Nv.x * Nv.y * Nv.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NT) return;
  int c[3];
  znew[g] = interior_of<DIM>(g, Nv, c) ? z[g] + (r[g] - stencil_apply<DIM>(A, z, g, Nv, NT)) / dl[g] : 0.0;
}
// rc = P^T s (2:1 vertex-centred): coarse I gathers fine 2I-1..2I+1 per axis with 1/2,1,1/2
template <int DIM>
__global__ void k_restrict_grid(const double* __restrict__ s, double* __restrict__ rc, int3 Nf, int3 Nc) {
  const long long NT = (long long)Nc.x * Nc.y * Nc.z;
  const long long I = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (I >= NT) return;
  int c[3];
  if (!interior_of<DIM>(I, Nc, c)) { rc[I] = 0.0; return; }
  double acc = 0.0;
  for (int oz = (DIM == 3 ? -1 : 0); oz <= (DIM == 3 ? 1 : 0); ++oz)
    for (int oy = -1; oy <= 1; ++oy)
      for (int ox = -1; ox <= 1; ++ox) {
        const double w = (ox ? 0.5 : 1.0) * (oy ? 0.5 : 1.0) * (oz ? 0.5 : 1.0);
        const long long f = (2 * c[0] + ox) + (long long)Nf.x * ((2 * c[1] + oy) + (long long)Nf.y * (DIM == 3 ? 2 * c[2] + oz : 0));
        acc += w * s[f];
      }
  rc[I] = acc;
}
// z += P e (2:1 vertex-centred), interior fine nodes only
template <int DIM>
__global__ void k_prolong_grid_add(const double* __restrict__ e, double* __restrict__ z, int3 Nf, int3 Nc) {
  const long long NT = (long long)Nf.x * Nf.y * Nf.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NT) return;
  int c[3];
  if (!interior_of<DIM>(g, Nf, c)) return;
  double acc = 0.0;
  for (int sel = 0; sel < (1 << DIM); ++sel) {
    double w = 1.0;
    int cc[3] = {0, 0, 0};
    bool ok = true;
    for (int k = 0; k < DIM; ++k) {
      const int b = (sel >> k) & 1;
      if (c[k] % 2 == 0) { if (b) { ok = false; break; } cc[k] = c[k] / 2; }
      else { cc[k] = c[k] / 2 + b; w *= 0.5; }
    }
    if (!ok) continue;
    acc += w * e[cc[0] + (long long)Nc.x * (cc[1] + (long long)Nc.y * cc[2])];
  }
  z[g] += acc;
}
// coarsest GMG level: dense LDL^T over its interior nodes (one block)
template <int DIM>
__global__ void k_coarsest_factor(const double* __restrict__ A, double* __restrict__ F, int3 Nv, int nint) {
  constexpr int ND = Dirs<DIM>::ND;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long NT = (long long)Nv.x * Nv.y * Nv.z;
  // interior index map
  int idx = 0;
  for (long long g = 0; g < NT; ++g) {
    int c[3];
    if (!interior_of<DIM>(g, Nv, c)) continue;
    for (int j = 0; j < nint; ++j) F[idx * nint + j] = 0.0;
    for (int d = 0; d < ND; ++d) {
      const long long h = g + dir_dx(d) + (long long)Nv.x * (dir_dy(d) + (long long)Nv.y * (DIM == 3 ? dir_dz(d) : 0));
      int cc[3];
      if (h < 0 || h >= NT || !interior_of<DIM>(h, Nv, cc)) continue;
      // interior rank of h
      int rk = 0;
      for (long long t = 0; t < h; ++t) { int c2[3]; if (interior_of<DIM>(t, Nv, c2)) ++rk; }
      F[idx * nint + rk] = A[(long long)d * NT + g];
    }
    ++idx;
  }
  // in-place Cholesky (lower)
  for (int j = 0; j < nint; ++j) {
    double s = F[j * nint + j];
    for (int k = 0; k < j; ++k) s -= F[j * nint + k] * F[j * nint + k];
    const double c = sqrt(s);
    F[j * nint + j] = c;
    for (int i = j + 1; i < nint; ++i) {
      double t = F[i * nint + j];
      for (int k = 0; k < j; ++k) t -= F[i * nint + k] * F[j * nint + k];
      F[i * nint + j] = t / c;
    }
  }
}
template <int DIM>
__global__ void k_coarsest_solve(const double* __restrict__ F, const double* __restrict__ r, double* __restrict__ z,
                                 int3 Nv, int nint) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long NT = (long long)Nv.x * Nv.y * Nv.z;
  double x[64];
  int idx = 0;
  for (long long g = 0; g < NT; ++g) { int c[3]; if (interior_of<DIM>(g, Nv, c)) x[idx++] = r[g]; }
  for (int i = 0; i < nint; ++i) {
    double s = x[i];
    for (int k = 0; k < i; ++k) s -= F[i * nint + k] * x[k];
    x[i] = s / F[i * nint + i];
  }
  for (int i = nint - 1; i >= 0; --i) {
    double s = x[i];
    for (int k = i + 1; k < nint; ++k) s -= F[k * nint + i] * x[k];
    x[i] = s / F[i * nint + i];
  }
  idx = 0;
  for (long long g = 0; g < NT; ++g) { int c[3]; z[g] = interior_of<DIM>(g, Nv, c) ? x[idx++] : 0.0; }
}

static inline unsigned nb(long long n, int t) { return (unsigned)((n + t - 1) / t); }
static inline int3 i3(const int* a) { return make_int3(a[0], a[1], a[2]); }

// ------------------------------------------------------------------ setup driver
static PatchGeom make_geom(const lorpc_prec* b) {
  PatchGeom G{};
  const lorpc_mesh* m = b->m;
  G.d = m->d; G.kind = b->desc.patch_kind; G.L = b->lor->L;
  for (int k = 0; k < 3; ++k) G.n[k] = m->n[k];
  for (int l = 0; l < G.L; ++l) {
    G.ml[l] = b->lor->ml[l];
    for (int k = 0; k < 3; ++k) G.Nax[l][k] = b->lor->Nax[l][k];
  }
  return G;
}

int schwarz_build(lorpc_prec* b, cudaStream_t s) {
  const lorpc_mesh* m = b->m;
  const lorpc_lor* lor = b->lor;
  const int d = m->d, L = lor->L, ND = d == 2 ? 9 : 27;
  b->L = L;
  PatchGeom G = make_geom(b);
  if (b->desc.patch_kind == 0) b->J = (long long)(m->n[0] + 1) * (m->n[1] + 1) * (d == 3 ? m->n[2] + 1 : 1);
  else b->J = m->nel;
  // record offsets (host; patch sizes are index arithmetic)
  b->recoff_h.assign((size_t)b->J * L, 0);
  long long off = 0;
  for (int l = 0; l < MAXL; ++l) b->max_n[l] = 0;
  for (long long j = 0; j < b->J; ++j)
    for (int l = 0; l < L; ++l) {
      int lo[3], ext[3];
      patch_box(G, j, l, lo, ext);
      const int n = std::max(ext[0] * ext[1] * ext[2], 0);
      if (n > 65535) return fail(LORPC_ERR_SIZE, "patch too large");
      b->max_n[l] = std::max(b->max_n[l], n);
      b->recoff_h[j * L + l] = off;
      off += rec_layout(n, num_edges(d, ext)).total;
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
  const long long per_warp = (long long)maxn * (2 * ND + 1) * 8 + (4ll * maxn + 1) * 4 + maxn;
  nwarps = std::max<long long>(1, std::min<long long>(nwarps, (2ll << 30) / per_warp));
  MdfParams P{};
  P.G = G;
  for (int l = 0; l < L; ++l) P.A[l] = lor->A[l];
  P.rec = b->rec; P.recoff = b->recoff; P.ntasks = ntasks; P.ordering = b->desc.ordering; P.maxn = maxn;
  LORPC_TRY(dalloc(&P.scratch, (size_t)nwarps * maxn * (2 * ND + 1)));
  LORPC_TRY(dalloc(&P.iscratch, (size_t)nwarps * (4 * maxn + 1)));
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
  // coarse space hierarchy (reading c11): level 0 = last LOR level (vertex grid)
  b->nc = 0;
  for (int i = 0; i < MAXC; ++i) { b->Ac[i] = b->dl1[i] = b->cr[i] = b->cz[i] = b->cs[i] = nullptr; }
  if (b->desc.coarse == 0) {
    int cur[3] = {m->n[0] + 1, m->n[1] + 1, d == 3 ? m->n[2] + 1 : 1};
    b->Ac[0] = lor->A[L - 1];
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
      LORPC_TRY(dalloc(&b->Ac[lvl + 1], (size_t)ND * Nn));
      int ne[3] = {nxt[0] - 1, nxt[1] - 1, nxt[2] - 1};
      LORPC_TRY(galerkin(d, b->Ac[lvl], b->Ac[lvl + 1], gmg_transfer(), ne, cur, nxt, s));
      for (int k = 0; k < 3; ++k) cur[k] = nxt[k];
      ++lvl;
    }
    b->nc = lvl + 1;
    // coarsest: dense Cholesky over its interior nodes
    int nint = 1;
    for (int k = 0; k < d; ++k) nint *= b->cn[lvl][k] - 2;
    if (nint > 64) return fail(LORPC_ERR_SIZE, "coarsest GMG level too large");
    b->ncoarsest = nint;
    LORPC_TRY(dalloc(&b->coarse_chol, (size_t)std::max(nint * nint, 1)));
    if (nint > 0) {
      if (d == 2) k_coarsest_factor<2><<<1, 1, 0, s>>>(b->Ac[lvl], b->coarse_chol, i3(b->cn[lvl]), nint);
      else k_coarsest_factor<3><<<1, 1, 0, s>>>(b->Ac[lvl], b->coarse_chol, i3(b->cn[lvl]), nint);
      LORPC_LAUNCHED();
    }
  }
  LORPC_CUDA(cudaStreamSynchronize(s));
  return LORPC_OK;
}

// ------------------------------------------------------------------ apply driver
template <int DIM>
static int coarse_apply(const lorpc_prec* b, const double* r, double* z, cudaStream_t s) {
  const lorpc_mesh* m = b->m;
  int3 nv = make_int3(m->n[0] + 1, m->n[1] + 1, DIM == 3 ? m->n[2] + 1 : 1);
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  k_restrict_vertex<DIM><<<nb(b->cN[0], 128), 128, 0, s>>>(r, b->cr[0], nv, N, m->basis);
  LORPC_LAUNCHED();
  const int K = b->nc - 1;
  for (int l = 0; l < K; ++l) {
    int3 Nv = i3(b->cn[l]), Nc = i3(b->cn[l + 1]);
    k_jacobi_pre<DIM><<<nb(b->cN[l], 256), 256, 0, s>>>(b->cr[l], b->dl1[l], b->cz[l], Nv);
    LORPC_LAUNCHED();
    k_residual_grid<DIM><<<nb(b->cN[l], 256), 256, 0, s>>>(b->Ac[l], b->cr[l], b->cz[l], b->cs[l], Nv);
    LORPC_LAUNCHED();
    k_restrict_grid<DIM><<<nb(b->cN[l + 1], 256), 256, 0, s>>>(b->cs[l], b->cr[l + 1], Nv, Nc);
    LORPC_LAUNCHED();
  }
  if (b->ncoarsest > 0) {
    k_coarsest_solve<DIM><<<1, 1, 0, s>>>(b->coarse_chol, b->cr[K], b->cz[K], i3(b->cn[K]), b->ncoarsest);
    LORPC_LAUNCHED();
  } else {
    LORPC_CUDA(cudaMemsetAsync(b->cz[K], 0, sizeof(double) * b->cN[K], s));
  }
  // level results: coarsest in cz[K], finer levels (after post-smoothing) in cs[l]
  for (int l = K - 1; l >= 0; --l) {
    int3 Nv = i3(b->cn[l]), Nc = i3(b->cn[l + 1]);
    const double* ec = (l + 1 == K) ? b->cz[l + 1] : b->cs[l + 1];
    k_prolong_grid_add<DIM><<<nb(b->cN[l], 256), 256, 0, s>>>(ec, b->cz[l], Nv, Nc);
    LORPC_LAUNCHED();
    k_jacobi_post<DIM><<<nb(b->cN[l], 256), 256, 0, s>>>(b->Ac[l], b->cr[l], b->dl1[l], b->cz[l], b->cs[l], Nv);
    LORPC_LAUNCHED();
  }
  const double* z0 = (K == 0) ? b->cz[0] : b->cs[0];
  k_prolong_vertex_add<DIM><<<nb(m->ndof_cg, 256), 256, 0, s>>>(z0, z, nv, N, n, m->basis);
  LORPC_LAUNCHED();
  return LORPC_OK;
}

template <int DIM>
__global__ void k_zero_dir(double* z, int3 N) {
  const long long NT = (long long)N.x * N.y * N.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NT) return;
  const int c0 = (int)(g % N.x), c1 = (int)((g / N.x) % N.y), c2 = (int)(g / ((long long)N.x * N.y));
  bool dd = c0 == 0 || c0 == N.x - 1 || c1 == 0 || c1 == N.y - 1;
  if (DIM == 3) dd = dd || c2 == 0 || c2 == N.z - 1;
  if (dd) z[g] = 0.0;
}

int schwarz_apply_cg(const lorpc_prec* b, const double* r, double* z, cudaStream_t s) {
  const lorpc_mesh* m = b->m;
  const lorpc_lor* lor = b->lor;
  const int d = m->d, L = b->L;
  LORPC_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * m->ndof_cg, s));
  VcParams P{};
  P.G = make_geom(b);
  for (int l = 0; l < L; ++l) { P.A[l] = lor->A[l]; if (l + 1 < L) P.T[l] = lor->T[l]; }
  P.rec = b->rec; P.recoff = b->recoff; P.J = b->J; P.r = r; P.z = z;
  int acc = 0;
  for (int l = 0; l < L; ++l) { P.soff[l] = acc; acc += 3 * b->max_n[l]; }
  P.warp_doubles = acc;
  const int warps_per_block = 4;
  const size_t smem = (size_t)warps_per_block * acc * sizeof(double);
  const unsigned blocks = (unsigned)((b->J + warps_per_block - 1) / warps_per_block);
  if (d == 2) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_vcycle<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_vcycle<2><<<blocks, 32 * warps_per_block, smem, s>>>(P);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_vcycle<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_vcycle<3><<<blocks, 32 * warps_per_block, smem, s>>>(P);
  }
  LORPC_LAUNCHED();
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  if (b->desc.coarse == 0) {
    if (d == 2) LORPC_TRY(coarse_apply<2>(b, r, z, s)); else LORPC_TRY(coarse_apply<3>(b, r, z, s));
  } else {
    if (d == 2) k_zero_dir<2><<<nb(m->ndof_cg, 256), 256, 0, s>>>(z, N);
    else k_zero_dir<3><<<nb(m->ndof_cg, 256), 256, 0, s>>>(z, N);
    LORPC_LAUNCHED();
  }
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
