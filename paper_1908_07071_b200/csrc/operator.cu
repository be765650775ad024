// Matrix-free CG operator y = K_p x by sum factorisation (row a2; P:104,
// P:742, tab:complexity P:764: O(p^{d+1}) work and O(p^d) memory per element).
//
// Per element: gather the (p+1)^d tile (Dirichlet entries masked to 0) ->
// 1D B/D contractions to the q^d Gauss points (q = p+1) -> multiply by the
// symmetric G_q -> transposed contractions -> scatter-add (atomics; free
// nodes only).  3D: one thread per line of the tile, every contraction in registers,
// four transposes through shared memory (k_cg3); several elements per CTA.
// y_D = x_D (symmetric Dirichlet elimination) is written by the pre-pass.
#include "device.cuh"

namespace lorpc {

template <int DIM>
__global__ void k_pre(const double* __restrict__ x, double* __restrict__ y, int3 N) {
  // 32-bit index arithmetic (grids below 2^31 nodes, checked by cg_apply)
  const unsigned ndof = (unsigned)N.x * N.y * N.z;
  const unsigned g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ndof) return;
  const unsigned gxy = g / (unsigned)N.x;
  const int gx = (int)(g - gxy * N.x), gy = (int)(gxy % (unsigned)N.y), gz = (int)(gxy / (unsigned)N.y);
  bool d = gx == 0 || gx == N.x - 1 || gy == 0 || gy == N.y - 1;
  if (DIM == 3) d = d || gz == 0 || gz == N.z - 1;
  y[g] = d ? x[g] : 0.0;
}

// Shared-memory layout of one transposed quantity of one element (row a2): Q^3 values
// addressed a * SA + k * SK + b, element stride SE (doubles).  The strides are chosen
// (offline bank model, scalar 64-bit accesses, lanes x-fastest over Q x Q x EB) so
// that both the writer pattern (lanes (i, j) at i SA + k SK + j or j SA + k SK + i,
// fixed k) and the reader pattern (lanes (i, j) at i SA + j SK + b or j SA + i SK + b,
// fixed b) are free of bank conflicts for Q = 2, 4 and nearly so otherwise.
template <int Q> struct CgLay;
template <> struct CgLay<2> { static constexpr int SK = 3, SA = 6, SE = 12; };
template <> struct CgLay<3> { static constexpr int SK = 3, SA = 9, SE = 27; };
template <> struct CgLay<4> { static constexpr int SK = 5, SA = 20, SE = 80; };
template <> struct CgLay<5> { static constexpr int SK = 5, SA = 29, SE = 149; };
template <> struct CgLay<6> { static constexpr int SK = 7, SA = 42, SE = 252; };
template <> struct CgLay<7> { static constexpr int SK = 9, SA = 63, SE = 441; };

// one element's threads sync: its Q^2 threads lie in one warp when Q^2 divides 32
template <int Q>
__device__ __forceinline__ void cg_sync() {
  if constexpr (32 % (Q * Q) == 0) __syncwarp(); else __syncthreads();
}

// 256-bit read-only load of four consecutive doubles (32-byte aligned)
__device__ __forceinline__ void ldg256(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}

// 3D operator, line-per-thread sum factorisation.  Thread (i, j) of an element owns a
// whole line of Q values in the direction being contracted, so every 1D contraction
// runs in registers with the basis matrices read as constant-bank operands
// (compile-time indices into the kernel parameter), and the data moves between the
// three line orientations by four transposes through shared memory (each value is
// written once and read once: 10 Q values per thread in, 10 Q out, against 22 Q
// reads of the stage-per-direction form):
//   z-lines at the nodes (a, b): u -> Bz u, Dz u                        [T1: -> y-lines]
//   y-lines (a, qz): -> By Bz u, Dy Bz u, By Dz u                       [T2: -> x-lines]
//   x-lines at the points (qy, qz): gradient, times G_q (one 256-bit load per
//     component when Q = 4), transposed x contraction                   [T2^T]
//   y-lines: transposed y contraction                                   [T1^T]
//   z-lines: transposed z contraction, scatter-add (atomics; free nodes only).
#ifndef LORPC_CG3_MINB
#define LORPC_CG3_MINB 6  // CTAs per SM asked of ptxas at p = 3 (measured on C5: 6 -> 1.64 ms, 7 (72 registers, spills) -> 1.88 ms, 8 -> 2.04 ms)
#endif
template <int P, int EB>
__global__ void __launch_bounds__((P + 1) * (P + 1) * EB, (P == 3 ? LORPC_CG3_MINB : 1))
k_cg3(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ G, int3 n, int3 N,
      const __grid_constant__ Basis1D bs, long long e0, long long e1, double* __restrict__ xy_part) {
  constexpr int Q = P + 1, Q2 = Q * Q, Q3 = Q * Q * Q;
  constexpr int SK = CgLay<Q>::SK, SA = CgLay<Q>::SA, SE = CgLay<Q>::SE;
  __shared__ double S[2][3][EB * SE];
  const int ti = threadIdx.x, tj = threadIdx.y, te = threadIdx.z;
  const long long e = e0 + (long long)blockIdx.x * EB + te;  // elements [e0, e1) (slab layers)
  const bool active = e < e1;
  int ex = 0, ey = 0, ez = 0;
  if (active) { ex = (int)(e % n.x); ey = (int)((e / n.x) % n.y); ez = (int)(e / ((long long)n.x * n.y)); }
  const int gx = ex * P + ti, gy = ey * P + tj;
  const bool bxy = gx == 0 || gx == N.x - 1 || gy == 0 || gy == N.y - 1;
  const long long base = gx + (long long)N.x * gy;
  const long long sz = (long long)N.x * N.y;
  // form-1 addresses (writer i SA + k SK + j, reader i SA + j SK + b), form 2 with i, j swapped
  double* const A0 = &S[0][0][te * SE];
  double* const B0 = &S[1][0][te * SE];
  constexpr int SQ = EB * SE;  // quantity stride
  const int w1 = ti * SA + tj, r1 = ti * SA + tj * SK;
  const int w2 = tj * SA + ti, r2 = tj * SA + ti * SK;

  // z-lines at the nodes (a = ti, b = tj)
  double u[Q];
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    const int gz = ez * P + c;
    const bool dir = bxy || gz == 0 || gz == N.z - 1;
    u[c] = (active && !dir) ? x[base + sz * gz] : 0.0;
  }
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double bu = 0.0, du = 0.0;
#pragma unroll
    for (int c = 0; c < Q; ++c) { bu += bs.B[qz * Q + c] * u[c]; du += bs.D[qz * Q + c] * u[c]; }
    A0[w1 + qz * SK] = bu;
    A0[SQ + w1 + qz * SK] = du;
  }
  cg_sync<Q>();
  // y-lines (a = ti, qz = tj)
  double v0[Q], v1[Q], v2[Q];
#pragma unroll
  for (int b = 0; b < Q; ++b) { v0[b] = A0[r1 + b]; v1[b] = A0[SQ + r1 + b]; }
#pragma unroll
  for (int qy = 0; qy < Q; ++qy) {
    double bb = 0.0, db = 0.0, bd = 0.0;
#pragma unroll
    for (int b = 0; b < Q; ++b) {
      bb += bs.B[qy * Q + b] * v0[b]; db += bs.D[qy * Q + b] * v0[b]; bd += bs.B[qy * Q + b] * v1[b];
    }
    B0[w2 + qy * SK] = bb;           // By Bz u  (-> Dx: d/dx)
    B0[SQ + w2 + qy * SK] = db;      // Dy Bz u  (-> Bx: d/dy)
    B0[2 * SQ + w2 + qy * SK] = bd;  // By Dz u  (-> Bx: d/dz)
  }
  cg_sync<Q>();
  // x-lines at the quadrature points (qy = ti, qz = tj)
#pragma unroll
  for (int a = 0; a < Q; ++a) { v0[a] = B0[r2 + a]; v1[a] = B0[SQ + r2 + a]; v2[a] = B0[2 * SQ + r2 + a]; }
  double f0[Q], f1[Q], f2[Q];
  {
    const double* Ge = G + (active ? e : 0) * 6 * Q3 + Q * (ti + Q * tj);
    double g[6][Q];
    if constexpr (Q == 4) {
#pragma unroll
      for (int c = 0; c < 6; ++c) ldg256(Ge + c * Q3, g[c]);
    } else {
#pragma unroll
      for (int c = 0; c < 6; ++c)
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) g[c][qx] = __ldg(Ge + c * Q3 + qx);
    }
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      double gxv = 0.0, gyv = 0.0, gzv = 0.0;
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        gxv += bs.D[qx * Q + a] * v0[a]; gyv += bs.B[qx * Q + a] * v1[a]; gzv += bs.B[qx * Q + a] * v2[a];
      }
      f0[qx] = g[0][qx] * gxv + g[1][qx] * gyv + g[2][qx] * gzv;
      f1[qx] = g[1][qx] * gxv + g[3][qx] * gyv + g[4][qx] * gzv;
      f2[qx] = g[2][qx] * gxv + g[4][qx] * gyv + g[5][qx] * gzv;
    }
  }
  // transposed x contraction (same lines), then to y-lines
#pragma unroll
  for (int a = 0; a < Q; ++a) {
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      p0 += bs.D[qx * Q + a] * f0[qx]; p1 += bs.B[qx * Q + a] * f1[qx]; p2 += bs.B[qx * Q + a] * f2[qx];
    }
    A0[w2 + a * SK] = p0;
    A0[SQ + w2 + a * SK] = p1;
    A0[2 * SQ + w2 + a * SK] = p2;
  }
  cg_sync<Q>();
  // y-lines (a = ti, qz = tj): transposed y contraction
#pragma unroll
  for (int qy = 0; qy < Q; ++qy) { v0[qy] = A0[r2 + qy]; v1[qy] = A0[SQ + r2 + qy]; v2[qy] = A0[2 * SQ + r2 + qy]; }
#pragma unroll
  for (int b = 0; b < Q; ++b) {
    double t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      t1 += bs.B[qy * Q + b] * v0[qy] + bs.D[qy * Q + b] * v1[qy];
      t2 += bs.B[qy * Q + b] * v2[qy];
    }
    B0[w1 + b * SK] = t1;       // (-> Bz^T)
    B0[SQ + w1 + b * SK] = t2;  // (-> Dz^T)
  }
  cg_sync<Q>();
  // z-lines at the nodes (a = ti, b = tj): transposed z contraction and scatter
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) { v0[qz] = B0[r1 + qz]; v1[qz] = B0[SQ + r1 + qz]; }
  // x . (K x) over the free nodes = the sum over the elements of x_e . (K_e x_e) (the masked
  // entries of u are zero): PCG's p . q leaves with the operator, one partial per CTA
  double xy = 0.0;
  if (active && !bxy) {
#pragma unroll
    for (int c = 0; c < Q; ++c) {
      const int gz = ez * P + c;
      if (gz == 0 || gz == N.z - 1) continue;
      double v = 0.0;
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) v += bs.B[qz * Q + c] * v0[qz] + bs.D[qz * Q + c] * v1[qz];
      atomicAdd(y + base + sz * gz, v);
      xy += u[c] * v;
    }
  }
  if (xy_part == nullptr) return;  // kernel-uniform
  xy = warp_sum(xy);
  __shared__ double red[(Q2 * EB + 31) / 32];
  const int lt = ti + Q * (tj + Q * te);
  if ((lt & 31) == 0) red[lt >> 5] = xy;
  __syncthreads();
  if (lt == 0) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < (Q2 * EB + 31) / 32; ++k) t += red[k];
    xy_part[blockIdx.x] = t;
  }
}

template <int P, int EB>
__global__ void __launch_bounds__((P + 1) * (P + 1) * EB)
k_cg2(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ G, int3 n, int3 N,
      Basis1D bs) {
  constexpr int Q = P + 1, Q2 = Q * Q;
  __shared__ double sB[Q2], sD[Q2];
  __shared__ double S[EB][2][Q2];
  const int tx = threadIdx.x, ty = threadIdx.y, te = threadIdx.z;
  const int lt = tx + Q * (ty + Q * te);
  for (int i = lt; i < Q2; i += Q2 * EB) { sB[i] = bs.B[i]; sD[i] = bs.D[i]; }
  const long long nel = (long long)n.x * n.y;
  const long long e = (long long)blockIdx.x * EB + te;
  const bool active = e < nel;
  int ex = 0, ey = 0;
  if (active) { ex = (int)(e % n.x); ey = (int)(e / n.x); }
  const int gx = ex * P + tx, gy = ey * P + ty;
  const bool dir = gx == 0 || gx == N.x - 1 || gy == 0 || gy == N.y - 1;
  const long long gi = gx + (long long)N.x * gy;
  double* S0 = S[te][0];
  double* S1 = S[te][1];
  S0[ty * Q + tx] = (active && !dir) ? x[gi] : 0.0;  // u[b][a]
  __syncthreads();
  // x contraction: thread (qx = tx, b = ty)
  double bx = 0.0, dx = 0.0;
#pragma unroll
  for (int a = 0; a < Q; ++a) { const double v = S0[ty * Q + a]; bx += sB[tx * Q + a] * v; dx += sD[tx * Q + a] * v; }
  __syncthreads();
  S0[ty * Q + tx] = bx; S1[ty * Q + tx] = dx;  // [b][qx]
  __syncthreads();
  // y contraction: thread (qx = tx, qy = ty)
  double gxv = 0.0, gyv = 0.0;
#pragma unroll
  for (int b = 0; b < Q; ++b) { gxv += sB[ty * Q + b] * S1[b * Q + tx]; gyv += sD[ty * Q + b] * S0[b * Q + tx]; }
  const int iq = tx + Q * ty;
  const double* Ge = G + (active ? e : 0) * 3 * Q2;
  const double g00 = Ge[iq], g01 = Ge[Q2 + iq], g11 = Ge[2 * Q2 + iq];
  const double fx = g00 * gxv + g01 * gyv, fy = g01 * gxv + g11 * gyv;
  __syncthreads();
  S0[ty * Q + tx] = fx; S1[ty * Q + tx] = fy;  // [qy][qx]
  __syncthreads();
  // y^T: thread (qx = tx, b = ty)
  double w1 = 0.0, w2 = 0.0;
#pragma unroll
  for (int qy = 0; qy < Q; ++qy) { w1 += sB[qy * Q + ty] * S0[qy * Q + tx]; w2 += sD[qy * Q + ty] * S1[qy * Q + tx]; }
  __syncthreads();
  S0[ty * Q + tx] = w1; S1[ty * Q + tx] = w2;  // [b][qx]
  __syncthreads();
  // x^T: thread (a = tx, b = ty)
  double v = 0.0;
#pragma unroll
  for (int qx = 0; qx < Q; ++qx) v += sD[qx * Q + tx] * S0[ty * Q + qx] + sB[qx * Q + tx] * S1[ty * Q + qx];
  if (active && !dir) atomicAdd(y + gi, v);
}

template <int P>
static void launch3(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s, double* xy_part) {
  constexpr int Q = P + 1;
  constexpr int EB = (Q * Q <= 16) ? 8 : (Q * Q <= 25 ? 4 : 2);  // 6 EB SE doubles of shared memory <= 48 KB
  int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  dim3 blk(Q, Q, EB);
  const long long e0 = (long long)m->ez_lo * m->n[0] * m->n[1], e1 = (long long)m->ez_hi * m->n[0] * m->n[1];
  unsigned grid = (unsigned)((e1 - e0 + EB - 1) / EB);
  if (grid == 0) return;
  k_cg3<P, EB><<<grid, blk, 0, s>>>(x, y, m->G, n, N, m->basis, e0, e1, xy_part);
}
template <int P>
static void launch2(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s) {
  constexpr int Q = P + 1;
  constexpr int EB = (Q * Q <= 16) ? 16 : (Q * Q <= 36 ? 8 : 4);
  int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  dim3 blk(Q, Q, EB);
  unsigned grid = (unsigned)((m->nel + EB - 1) / EB);
  k_cg2<P, EB><<<grid, blk, 0, s>>>(x, y, m->G, n, N, m->basis);
}

// CTAs of the 3D operator kernel (= partial sums of x . y it can write)
long long cg3_blocks(const lorpc_mesh* m) {
  if (m->d != 3) return 0;
  const int Q = m->p + 1;
  const int EB = (Q * Q <= 16) ? 8 : (Q * Q <= 25 ? 4 : 2);
  const long long ne = (long long)(m->ez_hi - m->ez_lo) * m->n[0] * m->n[1];
  return (ne + EB - 1) / EB;
}

// y = K x.  pre = false: y already holds x at the Dirichlet nodes and 0 elsewhere (the
// caller fused that pass).  xy_part != nullptr (3D only): cg3_blocks(m) partial sums of
// x . y over the free nodes.
int cg_apply_ex(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s, bool pre, double* xy_part) {
  if (m->ndof_cg >= (1ll << 31)) return fail(LORPC_ERR_SIZE, "cg_apply: grid of 2^31 nodes or more");
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  if (xy_part && m->d != 3) return fail(LORPC_ERR_ARG, "cg_apply: fused x . y is 3D only");
  if (pre) {
    const unsigned g = (unsigned)((m->ndof_cg + 255) / 256);
    if (m->d == 2) k_pre<2><<<g, 256, 0, s>>>(x, y, N); else k_pre<3><<<g, 256, 0, s>>>(x, y, N);
    LORPC_LAUNCHED();
  }
  if (m->d == 2) {
    switch (m->p) {
      case 1: launch2<1>(m, x, y, s); break; case 2: launch2<2>(m, x, y, s); break;
      case 3: launch2<3>(m, x, y, s); break; case 4: launch2<4>(m, x, y, s); break;
      case 5: launch2<5>(m, x, y, s); break; case 6: launch2<6>(m, x, y, s); break;
      case 7: launch2<7>(m, x, y, s); break; case 8: launch2<8>(m, x, y, s); break;
      default: return fail(LORPC_ERR_SIZE, "cg_apply: p not compiled");
    }
  } else {
    switch (m->p) {
      case 1: launch3<1>(m, x, y, s, xy_part); break; case 2: launch3<2>(m, x, y, s, xy_part); break;
      case 3: launch3<3>(m, x, y, s, xy_part); break; case 4: launch3<4>(m, x, y, s, xy_part); break;
      case 5: launch3<5>(m, x, y, s, xy_part); break; case 6: launch3<6>(m, x, y, s, xy_part); break;
      default: return fail(LORPC_ERR_SIZE, "cg_apply: p not compiled");
    }
  }
  LORPC_LAUNCHED();
  return LORPC_OK;
}

int cg_apply(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s) {
  return cg_apply_ex(m, x, y, s, true, nullptr);
}

}  // namespace lorpc
