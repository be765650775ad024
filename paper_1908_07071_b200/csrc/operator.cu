// Matrix-free CG operator y = K_p x by sum factorisation (row a2; P:104,
// P:742, tab:complexity P:764: O(p^{d+1}) work and O(p^d) memory per element).
//
// Per element: gather the (p+1)^d tile (Dirichlet entries masked to 0) ->
// 1D B/D contractions to the q^d Gauss points (q = p+1) -> multiply by the
// symmetric G_q -> transposed contractions -> scatter-add (atomics; free
// nodes only).  3D: one thread per (x,y) column of the tile, z contractions in
// registers, x/y contractions through shared memory; several elements per CTA.
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

// Q consecutive doubles from shared memory: 16-byte loads when Q is even (every read
// below starts at a multiple of Q doubles of a 16-byte-aligned array)
template <int Q>
__device__ __forceinline__ void lds_vec(const double* p, double (&v)[Q]) {
  if constexpr (Q % 2 == 0) {
#pragma unroll
    for (int i = 0; i < Q / 2; ++i) {
      const double2 t = reinterpret_cast<const double2*>(p)[i];
      v[2 * i] = t.x;
      v[2 * i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < Q; ++i) v[i] = p[i];
  }
}

template <int P, int EB>
__global__ void __launch_bounds__((P + 1) * (P + 1) * EB)
k_cg3(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ G, int3 n, int3 N,
      Basis1D bs, long long e0, long long e1) {
  constexpr int Q = P + 1, Q2 = Q * Q, Q3 = Q * Q * Q;
  __shared__ double sB[Q2], sD[Q2];
  // stage layouts: every contraction reads its Q operands contiguously (lds_vec)
  __shared__ __align__(16) double S[EB][3][Q3];
  const int tx = threadIdx.x, ty = threadIdx.y, te = threadIdx.z;
  const int lt = tx + Q * (ty + Q * te);
  for (int i = lt; i < Q2; i += Q2 * EB) { sB[i] = bs.B[i]; sD[i] = bs.D[i]; }
  const long long e = e0 + (long long)blockIdx.x * EB + te;  // elements [e0, e1) (slab layers)
  const bool active = e < e1;
  int ex = 0, ey = 0, ez = 0;
  if (active) { ex = (int)(e % n.x); ey = (int)((e / n.x) % n.y); ez = (int)(e / ((long long)n.x * n.y)); }
  const int gx = ex * P + tx, gy = ey * P + ty;
  const bool bxy = gx == 0 || gx == N.x - 1 || gy == 0 || gy == N.y - 1;
  const long long base = gx + (long long)N.x * gy;
  const long long sz = (long long)N.x * N.y;
  double u[Q];
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    const int gz = ez * P + c;
    const bool dir = bxy || gz == 0 || gz == N.z - 1;
    u[c] = (active && !dir) ? x[base + sz * gz] : 0.0;
  }
  __syncthreads();
  double* S0 = S[te][0];
  double* S1 = S[te][1];
  double* S2 = S[te][2];
  // z contraction (registers)
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double bu = 0.0, du = 0.0;
#pragma unroll
    for (int c = 0; c < Q; ++c) { bu += sB[qz * Q + c] * u[c]; du += sD[qz * Q + c] * u[c]; }
    S0[qz * Q2 + tx * Q + ty] = bu;  // [qz][a][b]
    S1[qz * Q2 + tx * Q + ty] = du;
  }
  __syncthreads();
  // y contraction: thread (a = tx, qy = ty)
  double r1[Q], r2[Q], r3[Q];
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double t1 = 0.0, t2 = 0.0, t3 = 0.0, v0[Q], v1[Q];
    lds_vec<Q>(S0 + qz * Q2 + tx * Q, v0);
    lds_vec<Q>(S1 + qz * Q2 + tx * Q, v1);
#pragma unroll
    for (int b = 0; b < Q; ++b) {
      t1 += sB[ty * Q + b] * v0[b]; t2 += sD[ty * Q + b] * v0[b]; t3 += sB[ty * Q + b] * v1[b];
    }
    r1[qz] = t1; r2[qz] = t2; r3[qz] = t3;
  }
  __syncthreads();
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    S0[qz * Q2 + ty * Q + tx] = r1[qz]; S1[qz * Q2 + ty * Q + tx] = r2[qz]; S2[qz * Q2 + ty * Q + tx] = r3[qz];
  }
  __syncthreads();
  // x contraction + geometric factors: thread (qx = tx, qy = ty)
  const double* Ge = G + (active ? e : 0) * 6 * Q3;
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double gxv = 0.0, gyv = 0.0, gzv = 0.0, v0[Q], v1[Q], v2[Q];
    lds_vec<Q>(S0 + qz * Q2 + ty * Q, v0);
    lds_vec<Q>(S1 + qz * Q2 + ty * Q, v1);
    lds_vec<Q>(S2 + qz * Q2 + ty * Q, v2);
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      gxv += sD[tx * Q + a] * v0[a];
      gyv += sB[tx * Q + a] * v1[a];
      gzv += sB[tx * Q + a] * v2[a];
    }
    const int iq = tx + Q * (ty + Q * qz);
    const double g00 = Ge[0 * Q3 + iq], g01 = Ge[1 * Q3 + iq], g02 = Ge[2 * Q3 + iq];
    const double g11 = Ge[3 * Q3 + iq], g12 = Ge[4 * Q3 + iq], g22 = Ge[5 * Q3 + iq];
    r1[qz] = g00 * gxv + g01 * gyv + g02 * gzv;
    r2[qz] = g01 * gxv + g11 * gyv + g12 * gzv;
    r3[qz] = g02 * gxv + g12 * gyv + g22 * gzv;
  }
  __syncthreads();
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    S0[qz * Q2 + ty * Q + tx] = r1[qz]; S1[qz * Q2 + ty * Q + tx] = r2[qz]; S2[qz * Q2 + ty * Q + tx] = r3[qz];
  }
  __syncthreads();
  // x^T: thread (a = tx, qy = ty)
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double w1 = 0.0, w2 = 0.0, w3 = 0.0, v0[Q], v1[Q], v2[Q];
    lds_vec<Q>(S0 + qz * Q2 + ty * Q, v0);
    lds_vec<Q>(S1 + qz * Q2 + ty * Q, v1);
    lds_vec<Q>(S2 + qz * Q2 + ty * Q, v2);
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      w1 += sD[qx * Q + tx] * v0[qx];
      w2 += sB[qx * Q + tx] * v1[qx];
      w3 += sB[qx * Q + tx] * v2[qx];
    }
    r1[qz] = w1; r2[qz] = w2; r3[qz] = w3;
  }
  __syncthreads();
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {  // [qz][a][qy]
    S0[qz * Q2 + tx * Q + ty] = r1[qz]; S1[qz * Q2 + tx * Q + ty] = r2[qz]; S2[qz * Q2 + tx * Q + ty] = r3[qz];
  }
  __syncthreads();
  // y^T: thread (a = tx, b = ty) -> YB (then B_z^T), YD (then D_z^T)
  double yb[Q], yd[Q];
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double t1 = 0.0, t2 = 0.0, v0[Q], v1[Q], v2[Q];
    lds_vec<Q>(S0 + qz * Q2 + tx * Q, v0);
    lds_vec<Q>(S1 + qz * Q2 + tx * Q, v1);
    lds_vec<Q>(S2 + qz * Q2 + tx * Q, v2);
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      t1 += sB[qy * Q + ty] * v0[qy] + sD[qy * Q + ty] * v1[qy];
      t2 += sB[qy * Q + ty] * v2[qy];
    }
    yb[qz] = t1; yd[qz] = t2;
  }
  // z^T and scatter
  if (!active || bxy) return;
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    const int gz = ez * P + c;
    if (gz == 0 || gz == N.z - 1) continue;
    double v = 0.0;
#pragma unroll
    for (int qz = 0; qz < Q; ++qz) v += sB[qz * Q + c] * yb[qz] + sD[qz * Q + c] * yd[qz];
    atomicAdd(y + base + sz * gz, v);
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
static void launch3(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s) {
  constexpr int Q = P + 1;
  constexpr int EB = (Q * Q <= 16) ? 8 : (Q * Q <= 36 ? 4 : 2);
  int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  dim3 blk(Q, Q, EB);
  const long long e0 = (long long)m->ez_lo * m->n[0] * m->n[1], e1 = (long long)m->ez_hi * m->n[0] * m->n[1];
  unsigned grid = (unsigned)((e1 - e0 + EB - 1) / EB);
  if (grid == 0) return;
  k_cg3<P, EB><<<grid, blk, 0, s>>>(x, y, m->G, n, N, m->basis, e0, e1);
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

int cg_apply(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s) {
  if (m->ndof_cg >= (1ll << 31)) return fail(LORPC_ERR_SIZE, "cg_apply: grid of 2^31 nodes or more");
  int3 N = make_int3(m->N[0], m->N[1], m->N[2]);
  const unsigned g = (unsigned)((m->ndof_cg + 255) / 256);
  if (m->d == 2) k_pre<2><<<g, 256, 0, s>>>(x, y, N); else k_pre<3><<<g, 256, 0, s>>>(x, y, N);
  LORPC_LAUNCHED();
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
      case 1: launch3<1>(m, x, y, s); break; case 2: launch3<2>(m, x, y, s); break;
      case 3: launch3<3>(m, x, y, s); break; case 4: launch3<4>(m, x, y, s); break;
      case 5: launch3<5>(m, x, y, s); break; case 6: launch3<6>(m, x, y, s); break;
      default: return fail(LORPC_ERR_SIZE, "cg_apply: p not compiled");
    }
  }
  LORPC_LAUNCHED();
  return LORPC_OK;
}

}  // namespace lorpc
