// Schwarz apply: patch V-cycles (rows a5, a6, a8) and the coarse correction (a7).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "patch.cuh"

#ifndef LORPC_VC_MINB
#define LORPC_VC_MINB 8   // min resident 128-thread blocks per SM for the V-cycle kernel
#endif

namespace lorpc {

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
// With rdot != nullptr the kernel also leaves per-block partial sums of r . z (the
// final z) in part[blockIdx.x]: PCG's rho = r.z fused into the last pass over z.
__device__ __forceinline__ double block_sum256(double v) {
  __shared__ double sh[8];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = threadIdx.x < 8 ? sh[threadIdx.x] : 0.0;
  if (w == 0) v = warp_sum(v);
  return v;
}
template <int DIM>
__device__ __forceinline__ double prolong_vertex_node(const double* __restrict__ zc, double* __restrict__ z, int3 nv,
                                                      int3 N, int3 n, const Basis1D& bs, unsigned g);
template <int DIM>
__global__ void __launch_bounds__(256) k_prolong_vertex_add(const double* __restrict__ zc, double* __restrict__ z, int3 nv,
                                                           int3 N, int3 n, Basis1D bs, const double* __restrict__ rdot,
                                                           double* __restrict__ part) {
  const unsigned NT = (unsigned)N.x * N.y * N.z;
  const unsigned g = blockIdx.x * blockDim.x + threadIdx.x;
  const double zg = g < NT ? prolong_vertex_node<DIM>(zc, z, nv, N, n, bs, g) : 0.0;
  if (rdot) {
    const double t = block_sum256(g < NT ? rdot[g] * zg : 0.0);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
  }
}
// z[g] += (P_0 zc)[g], z_D = 0; returns the new z[g]
template <int DIM>
__device__ __forceinline__ double prolong_vertex_node(const double* __restrict__ zc, double* __restrict__ z, int3 nv,
                                                      int3 N, int3 n, const Basis1D& bs, unsigned g) {
  // 32-bit index arithmetic (grids below 2^31 nodes, checked by the caller)
  const unsigned gxy = g / (unsigned)N.x;
  const int gc[3] = {(int)(g - gxy * N.x), (int)(gxy % (unsigned)N.y), (int)(gxy / (unsigned)N.y)};
  const int Nn[3] = {N.x, N.y, N.z}, nn[3] = {n.x, n.y, n.z};
  bool dir = false;
#pragma unroll
  for (int k = 0; k < DIM; ++k) if (gc[k] == 0 || gc[k] == Nn[k] - 1) dir = true;
  if (dir) { z[g] = 0.0; return 0.0; }
  const int p = bs.p;
  int v0[3] = {0, 0, 0};
  double w0[3] = {1, 1, 1}, w1[3] = {0, 0, 0};
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    const int e = min(gc[k] / p, nn[k] - 1);
    const int a = gc[k] - e * p;
    v0[k] = e; w1[k] = bs.xi[a]; w0[k] = 1.0 - w1[k];
  }
  double acc = 0.0;
  const unsigned vb = v0[0] + (unsigned)nv.x * (v0[1] + (unsigned)nv.y * v0[2]);
#pragma unroll
  for (int sel = 0; sel < (1 << DIM); ++sel) {
    double w = 1.0;
    unsigned off = 0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      const int b = (sel >> k) & 1;
      w *= b ? w1[k] : w0[k];
      if (b) off += k == 0 ? 1u : (k == 1 ? (unsigned)nv.x : (unsigned)nv.x * nv.y);
    }
    acc += w * __ldg(zc + vb + off);  // w = 0 terms read an existing vertex (clamped element)
  }
  const double zn = z[g] + acc;
  z[g] = zn;
  return zn;
}

// l1-Jacobi diagonal over interior columns of interior rows

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

// z = C^{-1} r on the coarsest interior (dense symmetric inverse, thread = row; the
// column walk makes the loads of a warp coalesced); boundary entries of z stay 0
__global__ void k_coarsest_inv(const double* __restrict__ Cinv, const int* __restrict__ idx,
                               const double* __restrict__ r, double* __restrict__ z, int nint) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nint) return;
  double acc = 0.0;
  for (int j = 0; j < nint; ++j) acc = fma(Cinv[(size_t)j * nint + i], __ldg(r + idx[j]), acc);
  z[idx[i]] = acc;
}

// ------------------------------------------------------------------ patch V-cycle
// VG = 8 lanes per patch, 4 patches per warp.  Shared memory per patch: the level
// vectors [r_l | z_l | s_l] for the finest levels, [r | z] at the dense level Ld,
// and a transfer scratch, addressed by 32-bit offsets into the dynamic array.
// ILU sweeps are row-per-lane: the rows of one DAG level (3-6 per patch on the
// MDF-ordered 3D patches) go to the lanes of the patch's group, each lane walks
// its row's entries; the next level's row data is prefetched into registers.
// Levels >= Ld (<= 32 free nodes per patch) are replaced by one precomputed dense
// symmetric matrix per patch, the exact operator of the V-cycle on those levels
// (k_dense_coarse builds it from the same ILU records).
constexpr int VG = 8, VPPW = 32 / VG;
extern __shared__ __align__(16) double vsm[];

struct VcParams {
  PatchGeom G;
  const double* A[MAXL];
  const double* W;        // separable 1D restriction tables (host-built, see schwarz.cu)
  int woff[MAXL][5];      // table offset for (level l -> l+1, elements along the axis 1..4)
  const char* rec;
  const long long* recoff;
  long long J;
  int Ld;                 // first level covered by the dense coarse operator
  double* Cd;             // [J][ldc] column-major n_Ld x n_Ld dense coarse V-cycle operators
  int ldc;
  int soff[MAXL];         // per-patch SMEM offsets (doubles) of [r | z | s] at level l
  int nmax[MAXL];
  int toff;               // transfer scratch offset
  int patch_doubles;
  const double* r;
  double* z;
};

// One triangular sweep of one patch level, DAG level by DAG level (reversed for
// the backward sweep): lane gl of the group takes rows lptr[lv] + gl, + VG, ...
// md = warp-uniform number of levels (max over the warp's patches).
__device__ __forceinline__ void sweep_rows(const double* __restrict__ Lv, const uint16_t* __restrict__ col,
                                           const uint16_t* __restrict__ rp, const uint16_t* __restrict__ sch,
                                           const uint16_t* __restrict__ lpt, int depth, int md, bool reverse, int v,
                                           int gl) {
  // prefetched row of the next level: node, entry range
  int prow = -1, pe0 = 0, pe1 = 0, pt = 0, pt1 = 0;
  auto fetch = [&](int it) {
    prow = -1;
    if (it >= depth) return;
    const int lv = reverse ? depth - 1 - it : it;
    pt = __ldg(lpt + lv) + gl;
    pt1 = __ldg(lpt + lv + 1);
    if (pt < pt1) { prow = __ldg(sch + pt); pe0 = __ldg(rp + pt); pe1 = __ldg(rp + pt + 1); }
  };
  fetch(0);
  for (int it = 0; it < md; ++it) {
    int row = prow, e0 = pe0, e1 = pe1, t = pt;
    const int t1 = pt1;
    fetch(it + 1);
    while (row >= 0) {
      double a0 = vsm[v + row], a1 = 0.0;
      int e = e0;
      for (; e + 3 < e1; e += 4) {
        const double l0 = __ldg(Lv + e), l1 = __ldg(Lv + e + 1), l2 = __ldg(Lv + e + 2), l3 = __ldg(Lv + e + 3);
        const int c0 = __ldg(col + e), c1 = __ldg(col + e + 1), c2 = __ldg(col + e + 2), c3 = __ldg(col + e + 3);
        a0 -= l0 * vsm[v + c0];
        a1 -= l1 * vsm[v + c1];
        a0 -= l2 * vsm[v + c2];
        a1 -= l3 * vsm[v + c3];
      }
      for (; e < e1; ++e) a0 -= __ldg(Lv + e) * vsm[v + __ldg(col + e)];
      vsm[v + row] = a0 + a1;
      // a level wider than VG rows: further rows of this lane
      t += VG;
      row = -1;
      if (t < t1) { row = __ldg(sch + t); e0 = __ldg(rp + t); e1 = __ldg(rp + t + 1); }
    }
    __syncwarp();
  }
}

// v := M^{-1} v, M = L D L^T of one patch level (forward L, diagonal, backward L^T)
__device__ __forceinline__ void ilu_w(const char* __restrict__ rec, bool act, int v, int gl) {
  int n = 0, depth = 0, nL = 0;
  if (act) { const int4 h = __ldg((const int4*)rec); n = h.x; depth = h.y; nL = h.z; }
  const int md = __reduce_max_sync(0xffffffffu, depth);
  if (md == 0) return;
  const RecLayout R = rec_layout(n, nL);
  const uint16_t* sch = (const uint16_t*)(rec + R.sched);
  const uint16_t* lpt = (const uint16_t*)(rec + R.lptr);
  sweep_rows((const double*)(rec + R.L), (const uint16_t*)(rec + R.nb), (const uint16_t*)(rec + R.frp), sch, lpt,
             depth, md, false, v, gl);
  const double* D = (const double*)(rec + R.D);
  for (int i = gl; i < n; i += VG) vsm[v + i] = vsm[v + i] / __ldg(D + i);
  __syncwarp();
  sweep_rows((const double*)(rec + R.bL), (const uint16_t*)(rec + R.bk), (const uint16_t*)(rec + R.brp), sch, lpt,
             depth, md, true, v, gl);
}

// s = r - A_l z on the patch box (A_l row-major: ND contiguous doubles per node)
template <int DIM>
__device__ __forceinline__ void residual_w(const double* __restrict__ A, long long Nx, long long Ny, long long NT, const int* lo,
                                           const int* ext, int r, int z, int s, int gl) {
  constexpr int ND = Dirs<DIM>::ND;
  const int ex = ext[0], ey = ext[1], ez = ext[2], n = ex * ey * ez;
  const float rex = 1.0f / ex, rexy = 1.0f / (ex * ey);
  for (int i = gl; i < n; i += VG) {
    int ix, iy, iz;
    box_xyz(i, ex, ey, rex, rexy, ix, iy, iz);
    const long long gi = (lo[0] + ix) + Nx * ((lo[1] + iy) + Ny * (DIM == 3 ? lo[2] + iz : 0));
    const double* Ar = A + gi * Dirs<DIM>::NDP;
    const uint32_t em = exist_mask<DIM>(ix, iy, iz, ex, ey, ez);
    double a0 = vsm[r + i], a1 = 0.0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const double zv = (em & (1u << d)) ? vsm[z + i + doff<DIM>(d, ex, ey)] : 0.0;
      const double t2 = __ldg(Ar + d) * zv;
      if (d & 1) a1 += t2; else a0 -= t2;
    }
    vsm[s + i] = a0 - a1;
  }
}

// rc = P^T s (separable: x, y, z passes through the scratch T at offset t)
template <int DIM>
__device__ __forceinline__ void restrict_w(const double* Wx, const double* Wy, const double* Wz, const int* ext,
                                           const int* cext, int s, int rc, int t, int gl) {
  const int fx = ext[0], fy = ext[1], fz = ext[2], cx = cext[0], cy = cext[1], cz = cext[2];
  const float rcx = 1.0f / max(cx, 1), rcxy = 1.0f / max(cx * cy, 1);
  const int T2 = DIM == 3 ? t + cx * fy * fz : rc;
  for (int u = gl; u < cx * fy * fz; u += VG) {
    const int rest = qdiv(u, rcx), ic = u - rest * cx;
    double a = 0.0;
    for (int f = 0; f < fx; ++f) a += __ldg(Wx + ic * fx + f) * vsm[s + f + fx * rest];
    vsm[t + u] = a;
  }
  __syncwarp();
  for (int u = gl; u < cx * cy * fz; u += VG) {
    const int kf = qdiv(u, rcxy), r2 = u - kf * cx * cy, jc = qdiv(r2, rcx), ic = r2 - jc * cx;
    double a = 0.0;
    for (int f = 0; f < fy; ++f) a += __ldg(Wy + jc * fy + f) * vsm[t + ic + cx * (f + fy * kf)];
    vsm[T2 + u] = a;
  }
  __syncwarp();
  if (DIM == 3) {
    for (int u = gl; u < cx * cy * cz; u += VG) {
      const int kc = qdiv(u, rcxy), ij = u - kc * cx * cy;
      double a = 0.0;
      for (int f = 0; f < fz; ++f) a += __ldg(Wz + kc * fz + f) * vsm[T2 + ij + cx * cy * f];
      vsm[rc + u] = a;
    }
    __syncwarp();
  }
}

// z += P e (separable transpose of restrict_w)
template <int DIM>
__device__ __forceinline__ void prolong_w(const double* Wx, const double* Wy, const double* Wz, const int* ext,
                                          const int* cext, int e, int z, int t, int gl) {
  const int fx = ext[0], fy = ext[1], fz = ext[2], cx = cext[0], cy = cext[1], cz = cext[2];
  const float rcx = 1.0f / max(cx, 1), rcxy = 1.0f / max(cx * cy, 1), rcxfy = 1.0f / max(cx * fy, 1),
              rfx = 1.0f / max(fx, 1);
  int U2 = e;
  if (DIM == 3) {
    U2 = t + cx * fy * fz;
    for (int u = gl; u < cx * cy * fz; u += VG) {           // z pass: [cx][cy][fz]
      const int kf = qdiv(u, rcxy), ij = u - kf * cx * cy;
      double a = 0.0;
      for (int c = 0; c < cz; ++c) a += __ldg(Wz + c * fz + kf) * vsm[e + ij + cx * cy * c];
      vsm[U2 + u] = a;
    }
    __syncwarp();
  }
  for (int u = gl; u < cx * fy * fz; u += VG) {             // y pass: [cx][fy][fz]
    const int kf = qdiv(u, rcxfy), r2 = u - kf * cx * fy, jf = qdiv(r2, rcx), ic = r2 - jf * cx;
    double a = 0.0;
    for (int c = 0; c < cy; ++c) a += __ldg(Wy + c * fy + jf) * vsm[U2 + ic + cx * (c + cy * kf)];
    vsm[t + u] = a;
  }
  __syncwarp();
  const int n = fx * fy * fz;
  for (int i = gl; i < n; i += VG) {                         // x pass, z += P e
    const int rest = qdiv(i, rfx), fxi = i - rest * fx;
    double a = 0.0;
    for (int c = 0; c < cx; ++c) a += __ldg(Wx + c * fx + fxi) * vsm[t + c + cx * rest];
    vsm[z + i] += a;
  }
  __syncwarp();
}

// Patch geometry of one group's patch
struct PatchCtx {
  int elo[3], ec[3];
  bool act;
};
template <int DIM>
__device__ __forceinline__ void box_of(const VcParams& P, const PatchCtx& c, int l, int* lo, int* ext) {
  const int m = P.G.ml[l];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (k >= DIM) { lo[k] = 0; ext[k] = 1; continue; }
    lo[k] = c.elo[k] * (m - 1) + 1;
    ext[k] = c.act ? c.ec[k] * (m - 1) - 1 : 0;
  }
}

// V(1,1) over levels l0..l1-1 with ILU smoothing; at level l1 either the dense
// operator (dense = true) or the ILU record (an exact solve at the coarsest level).
// Input r_{l0} at soff[l0], output z_{l0} at soff[l0] + nmax[l0].
template <int DIM>
__device__ void vcycle_range(const VcParams& P, const PatchCtx& c, long long j, int base, int l0, int l1, bool dense,
                             int gl) {
  const int L = P.G.L;
  auto rv = [&](int l) { return base + P.soff[l]; };
  auto zv = [&](int l) { return base + P.soff[l] + P.nmax[l]; };
  auto sv = [&](int l) { return base + P.soff[l] + 2 * P.nmax[l]; };
  auto recl = [&](int l) { return P.rec + (c.act ? P.recoff[j * L + l] : 0); };
  const int T = base + P.toff;
  for (int l = l0; l < l1; ++l) {
    int lo[3], ext[3], clo[3], cext[3];
    box_of<DIM>(P, c, l, lo, ext);
    box_of<DIM>(P, c, l + 1, clo, cext);
    const int n = ext[0] * ext[1] * ext[2];
    for (int i = gl; i < n; i += VG) vsm[zv(l) + i] = vsm[rv(l) + i];
    __syncwarp();
    ilu_w(recl(l), c.act, zv(l), gl);                          // pre-smoothing
    residual_w<DIM>(P.A[l], P.G.Nax[l][0], P.G.Nax[l][1], (long long)P.G.Nax[l][0] * P.G.Nax[l][1] * P.G.Nax[l][2], lo, ext, rv(l), zv(l), sv(l), gl);
    __syncwarp();
    restrict_w<DIM>(P.W + P.woff[l][c.ec[0]], P.W + P.woff[l][c.ec[1]], P.W + P.woff[l][DIM == 3 ? c.ec[2] : 1],
                    ext, cext, sv(l), rv(l + 1), T, gl);
  }
  {
    int lo[3], ext[3];
    box_of<DIM>(P, c, l1, lo, ext);
    const int n = ext[0] * ext[1] * ext[2];
    if (dense) {                                               // z = C r (column-major, symmetric)
      const double* C = P.Cd + (c.act ? j : 0) * (long long)P.ldc;
      for (int i = gl; i < n; i += VG) {
        double a0 = 0.0, a1 = 0.0;
        int k = 0;
        for (; k + 1 < n; k += 2) {
          a0 += __ldg(C + (long long)k * n + i) * vsm[rv(l1) + k];
          a1 += __ldg(C + (long long)(k + 1) * n + i) * vsm[rv(l1) + k + 1];
        }
        if (k < n) a0 += __ldg(C + (long long)k * n + i) * vsm[rv(l1) + k];
        vsm[zv(l1) + i] = a0 + a1;
      }
      __syncwarp();
    } else {
      for (int i = gl; i < n; i += VG) vsm[zv(l1) + i] = vsm[rv(l1) + i];
      __syncwarp();
      ilu_w(recl(l1), c.act, zv(l1), gl);
    }
  }
  for (int l = l1 - 1; l >= l0; --l) {
    int lo[3], ext[3], clo[3], cext[3];
    box_of<DIM>(P, c, l, lo, ext);
    box_of<DIM>(P, c, l + 1, clo, cext);
    const int n = ext[0] * ext[1] * ext[2];
    prolong_w<DIM>(P.W + P.woff[l][c.ec[0]], P.W + P.woff[l][c.ec[1]], P.W + P.woff[l][DIM == 3 ? c.ec[2] : 1],
                   ext, cext, zv(l + 1), zv(l), T, gl);
    residual_w<DIM>(P.A[l], P.G.Nax[l][0], P.G.Nax[l][1], (long long)P.G.Nax[l][0] * P.G.Nax[l][1] * P.G.Nax[l][2], lo, ext, rv(l), zv(l), sv(l), gl);
    __syncwarp();
    ilu_w(recl(l), c.act, sv(l), gl);                          // post-smoothing
    for (int i = gl; i < n; i += VG) vsm[zv(l) + i] += vsm[sv(l) + i];
    __syncwarp();
  }
}

template <int DIM>
__device__ __forceinline__ PatchCtx patch_ctx(const VcParams& P, long long j) {
  PatchCtx c;
  c.act = j < P.J;
  int ehi[3] = {0, 0, 0};
  c.elo[0] = c.elo[1] = c.elo[2] = 0;
  if (c.act) patch_elems(P.G, j, c.elo, ehi);
#pragma unroll
  for (int k = 0; k < 3; ++k) c.ec[k] = ehi[k] - c.elo[k] + 1;
  return c;
}

template <int DIM>
__global__ void __launch_bounds__(128, LORPC_VC_MINB) k_vcycle(VcParams P) {
  const int lane = threadIdx.x & 31, grp = lane / VG, gl = lane % VG;
  const long long wg = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (wg * VPPW >= P.J) return;  // warp-uniform
  const long long j = wg * VPPW + grp;
  const int base = ((threadIdx.x >> 5) * VPPW + grp) * P.patch_doubles;
  const PatchCtx c = patch_ctx<DIM>(P, j);
  int lo[3], ext[3];
  box_of<DIM>(P, c, 0, lo, ext);
  const int n = ext[0] * ext[1] * ext[2];
  const long long Nx = P.G.Nax[0][0], Ny = P.G.Nax[0][1];
  const float rex = 1.0f / max(ext[0], 1), rexy = 1.0f / max(ext[0] * ext[1], 1);
  for (int i = gl; i < n; i += VG) {                          // r_j = I_j^T r (a5)
    int ix, iy, iz;
    box_xyz(i, ext[0], ext[1], rex, rexy, ix, iy, iz);
    vsm[base + P.soff[0] + i] = __ldg(P.r + (lo[0] + ix) + Nx * ((lo[1] + iy) + Ny * (DIM == 3 ? lo[2] + iz : 0)));
  }
  __syncwarp();
  vcycle_range<DIM>(P, c, j, base, 0, P.Ld, true, gl);
  const int z0 = base + P.soff[0] + P.nmax[0];
  for (int i = gl; i < n; i += VG) {                          // z += I_j z_j (a8)
    int ix, iy, iz;
    box_xyz(i, ext[0], ext[1], rex, rexy, ix, iy, iz);
    atomicAdd(P.z + (lo[0] + ix) + Nx * ((lo[1] + iy) + Ny * (DIM == 3 ? lo[2] + iz : 0)), vsm[z0 + i]);
  }
}

// setup: dense operator of the V-cycle on levels Ld..L-1 for every patch (columns
// = images of the unit vectors); warp-uniform column loop
template <int DIM>
__global__ void __launch_bounds__(128) k_dense_coarse(VcParams P) {
  const int lane = threadIdx.x & 31, grp = lane / VG, gl = lane % VG;
  const long long wg = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (wg * VPPW >= P.J) return;
  const long long j = wg * VPPW + grp;
  const int base = ((threadIdx.x >> 5) * VPPW + grp) * P.patch_doubles;
  PatchCtx c = patch_ctx<DIM>(P, j);
  const int Ld = P.Ld, L = P.G.L;
  int lo[3], ext[3];
  box_of<DIM>(P, c, Ld, lo, ext);
  const int n = ext[0] * ext[1] * ext[2];
  const int nw = __reduce_max_sync(0xffffffffu, n);
  double* C = P.Cd + (c.act ? j : 0) * (long long)P.ldc;
  const bool act0 = c.act;
  for (int k = 0; k < nw; ++k) {
    c.act = act0 && k < n;
    for (int i = gl; i < n; i += VG) vsm[base + P.soff[Ld] + i] = (i == k) ? 1.0 : 0.0;
    __syncwarp();
    vcycle_range<DIM>(P, c, j, base, Ld, L - 1, false, gl);
    if (c.act)
      for (int i = gl; i < n; i += VG) C[(long long)k * n + i] = vsm[base + P.soff[Ld] + P.nmax[Ld] + i];
    __syncwarp();
  }
}

// ------------------------------------------------------------------ apply driver
// One GMG V(1,1) of R_0 (reading c11) on the hierarchy of gmg_build: input cr[0],
// result in *out (cz[0] or cs[0]).
template <int DIM>
static int gmg_vcycle_t(const lorpc_prec* b, const double** out, cudaStream_t s) {
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
    k_coarsest_inv<<<nb(b->ncoarsest, 128), 128, 0, s>>>(b->coarse_chol, b->coarse_idx, b->cr[K], b->cz[K],
                                                          b->ncoarsest);
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
  *out = (K == 0) ? b->cz[0] : b->cs[0];
  return LORPC_OK;
}
// z += P_0 zc on the mesh's node grid (zc on its vertex grid; Dirichlet nodes set to 0)
int prolong_vertex_add(const lorpc_mesh* m, const double* zc, double* z, cudaStream_t s) {
  int3 nv = make_int3(m->n[0] + 1, m->n[1] + 1, m->d == 3 ? m->n[2] + 1 : 1);
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]), n = make_int3(m->n[0], m->n[1], m->n[2]);
  if (m->ndof_cg >= (1ll << 31)) return fail(LORPC_ERR_SIZE, "prolong_vertex_add: grid of 2^31 nodes or more");
  if (m->d == 2) k_prolong_vertex_add<2><<<nb(m->ndof_cg, 256), 256, 0, s>>>(zc, z, nv, N, n, m->basis, nullptr, nullptr);
  else k_prolong_vertex_add<3><<<nb(m->ndof_cg, 256), 256, 0, s>>>(zc, z, nv, N, n, m->basis, nullptr, nullptr);
  LORPC_LAUNCHED();
  return LORPC_OK;
}
int gmg_vcycle(const lorpc_prec* b, const double** out, cudaStream_t s) {
  return b->m->d == 2 ? gmg_vcycle_t<2>(b, out, s) : gmg_vcycle_t<3>(b, out, s);
}

// R_0 part of B (a7), split so that P_0^T r and the GMG V-cycle run on the aux stream
// concurrently with the patch batch ("each of the local approximate solvers R_j
// may be applied in parallel"); the prolongation P_0 z_0 joins on s.
template <int DIM>
static int coarse_restrict_solve(const lorpc_prec* b, const double* r, const double** z0, cudaStream_t s) {
  const lorpc_mesh* m = b->m;
  int3 nv = make_int3(m->n[0] + 1, m->n[1] + 1, DIM == 3 ? m->n[2] + 1 : 1);
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  k_restrict_vertex<DIM><<<nb(b->cN[0], 128), 128, 0, s>>>(r, b->cr[0], nv, N, m->basis);
  LORPC_LAUNCHED();
  return gmg_vcycle_t<DIM>(b, z0, s);
}
template <int DIM>
static int coarse_prolong(const lorpc_prec* b, const double* z0, double* z, const double* rdot, double* part,
                          cudaStream_t s) {
  const lorpc_mesh* m = b->m;
  int3 nv = make_int3(m->n[0] + 1, m->n[1] + 1, DIM == 3 ? m->n[2] + 1 : 1);
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  if (m->ndof_cg >= (1ll << 31)) return fail(LORPC_ERR_SIZE, "coarse_apply: grid of 2^31 nodes or more");
  k_prolong_vertex_add<DIM><<<nb(m->ndof_cg, 256), 256, 0, s>>>(z0, z, nv, N, n, m->basis, rdot, part);
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

static VcParams make_params(const lorpc_prec* b, const double* r, double* z) {
  const lorpc_lor* lor = b->lor;
  const int L = b->L;
  VcParams P{};
  P.G = make_geom(b);
  for (int l = 0; l < L; ++l) P.A[l] = lor->A[l];
  P.W = b->wtab;
  memcpy(P.woff, b->woff, sizeof(P.woff));
  P.rec = b->rec; P.recoff = b->recoff; P.J = b->J; P.r = r; P.z = z;
  P.Ld = b->Ld; P.Cd = b->Cd; P.ldc = b->ldc;
  int acc = 0;
  for (int l = 0; l < L; ++l) { P.soff[l] = acc; P.nmax[l] = b->max_n[l]; acc += 3 * b->max_n[l]; }
  P.toff = acc;
  acc += b->scratch_doubles;
  P.patch_doubles = (acc + 1) & ~1;
  return P;
}

template <int DIM, bool SETUP>
static int launch_vc(const VcParams& P, long long J, cudaStream_t s) {
  const size_t per_warp = (size_t)VPPW * P.patch_doubles * sizeof(double);
  int wpb = 4;
  while (wpb > 1 && per_warp * wpb > 113 * 1024) wpb >>= 1;
  const size_t smem = per_warp * wpb;
  if (smem > 227 * 1024) return fail(LORPC_ERR_SIZE, "vcycle: patch does not fit in shared memory");
  const long long warps = (J + VPPW - 1) / VPPW;
  const unsigned blocks = (unsigned)((warps + wpb - 1) / wpb);
  if (SETUP) {
    cudaFuncSetAttribute(k_dense_coarse<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_dense_coarse<DIM><<<blocks, 32 * wpb, smem, s>>>(P);
  } else {
    cudaFuncSetAttribute(k_vcycle<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_vcycle<DIM><<<blocks, 32 * wpb, smem, s>>>(P);
  }
  LORPC_LAUNCHED();
  return LORPC_OK;
}

int vcycle_t_apply(const lorpc_prec* b, const double* r, double* z, cudaStream_t s);  // vcycle_t.cu
int vcycle_w_apply(const lorpc_prec* b, const double* r, double* z, cudaStream_t s);  // vcycle_w.cu
int vcycle_q_apply(const lorpc_prec* b, const double* r, double* z, cudaStream_t s);  // vcycle_w.cu

int dense_coarse_setup(lorpc_prec* b, cudaStream_t s) {
  VcParams P = make_params(b, nullptr, nullptr);
  return b->m->d == 2 ? launch_vc<2, true>(P, b->J, s) : launch_vc<3, true>(P, b->J, s);
}

// z = sum_j I_j B_j I_j^T r over the patches (no coarse term, z not zeroed at Dirichlet nodes)
int schwarz_apply_patches(const lorpc_prec* b, const double* r, double* z, cudaStream_t s) {
  LORPC_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * b->m->ndof_cg, s));
  if (b->qmode) return vcycle_q_apply(b, r, z, s);
  if (b->wmode) return vcycle_w_apply(b, r, z, s);
  if (b->tmode) return vcycle_t_apply(b, r, z, s);
  VcParams P = make_params(b, r, z);
  return b->m->d == 2 ? launch_vc<2, false>(P, b->J, s) : launch_vc<3, false>(P, b->J, s);
}

int single_apply(const lorpc_prec* b, const double* r, double* z, cudaStream_t s);  // single.cu

int schwarz_apply_cg(const lorpc_prec* b, const double* r, double* z, cudaStream_t s, double* rzpart) {
  const lorpc_mesh* m = b->m;
  const int d = m->d;
  if (b->desc.patch_kind == 2) {  // B(1): R_0 at the bottom of the one V-cycle, no additive term
    if (rzpart) return fail(LORPC_ERR_ARG, "schwarz_apply_cg: fused r.z needs the additive coarse term");
    return single_apply(b, r, z, s);
  }
  const bool coarse = b->desc.coarse == 0;
  const double* z0 = nullptr;
  // R_0 concurrently with the patch batch on the aux stream is opt-in (LORPC_OVERLAP=1):
  // measured on C5 it slows the thread-mode V-cycle from 42 to 60 ms per apply
  // (DESIGN.md 5.2), far more than the ~1 ms the R_0 chain takes serially
  static const int overlap = getenv("LORPC_OVERLAP") ? atoi(getenv("LORPC_OVERLAP")) : 0;
  if (coarse && overlap) {  // fork: R_0 chain on the aux stream
    LORPC_CUDA(cudaEventRecord(b->evf, s));
    LORPC_CUDA(cudaStreamWaitEvent(b->aux, b->evf, 0));
    if (d == 2) LORPC_TRY(coarse_restrict_solve<2>(b, r, &z0, b->aux));
    else LORPC_TRY(coarse_restrict_solve<3>(b, r, &z0, b->aux));
    LORPC_CUDA(cudaEventRecord(b->evj, b->aux));
  }
  LORPC_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * m->ndof_cg, s));
  VcParams P = make_params(b, r, z);
  lorpc_prec* bm = const_cast<lorpc_prec*>(b);
  const bool prof = bm->prof_on && bm->prof_n < (int)bm->prof_ev.size() / 2;
  if (prof) LORPC_CUDA(cudaEventRecord(bm->prof_ev[2 * bm->prof_n], s));
  const int rc = b->qmode ? vcycle_q_apply(b, r, z, s)
                 : b->wmode ? vcycle_w_apply(b, r, z, s)
                 : b->tmode ? vcycle_t_apply(b, r, z, s)
                 : d == 2 ? launch_vc<2, false>(P, b->J, s) : launch_vc<3, false>(P, b->J, s);
  if (rc != LORPC_OK) return rc;
  if (prof) { LORPC_CUDA(cudaEventRecord(bm->prof_ev[2 * bm->prof_n + 1], s)); bm->prof_n++; }
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  if (coarse) {  // join, then z += P_0 z_0 (and z_D = 0)
    if (overlap) {
      LORPC_CUDA(cudaStreamWaitEvent(s, b->evj, 0));
    } else if (d == 2) {
      LORPC_TRY(coarse_restrict_solve<2>(b, r, &z0, s));
    } else {
      LORPC_TRY(coarse_restrict_solve<3>(b, r, &z0, s));
    }
    if (d == 2) LORPC_TRY(coarse_prolong<2>(b, z0, z, rzpart ? r : nullptr, rzpart, s));
    else LORPC_TRY(coarse_prolong<3>(b, z0, z, rzpart ? r : nullptr, rzpart, s));
  } else {
    if (rzpart) return fail(LORPC_ERR_ARG, "schwarz_apply_cg: fused r.z needs the coarse term");
    if (d == 2) k_zero_dir<2><<<nb(m->ndof_cg, 256), 256, 0, s>>>(z, N);
    else k_zero_dir<3><<<nb(m->ndof_cg, 256), 256, 0, s>>>(z, N);
    LORPC_LAUNCHED();
  }
  return LORPC_OK;
}

}  // namespace lorpc
