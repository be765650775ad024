// Symmetric interior penalty DG (rows a3, a9; eq:ip P:113-136, eq:dg-as P:635-641).
//
// y = A_IP x = (grad u, grad v) - <{grad u},[v]> - <[u],{grad v}> + <sigma [u],[v]>,
// [phi] = phi^- n^- + phi^+ n^+, {phi} = (phi^- + phi^+)/2; boundary
// faces one-sided ([u] = u n, {grad u} = grad u; reading c15); sigma_e = eta/h_e,
// h_e = min(|K^-|,|K^+|)/|e| (readings c13, c14); Gauss q = p+1 on volumes and
// faces (reading c1).  DG vectors are element-major [n_el][(p+1)^3].
//
// Volume: the CG sum-factorised kernel on element-local dofs (plain stores).
// Faces: one CTA per face, one thread per face Gauss point.  With the GLL nodal
// basis the trace on a face only involves the face nodes, and the reference
// normal derivative is sum_a l_a'(end) u(a, .); both are reduced to two
// (p+1)^2 slabs per side and interpolated to the face points by 2D sum
// factorisation; the test-function side is the transpose.  Contributions are
// added with atomics after the volume pass.  3D only (config C4).
#include "device.cuh"

namespace lorpc {

// ----------------------------------------------------------------- volume term
template <int P, int EB>
__global__ void __launch_bounds__((P + 1) * (P + 1) * EB)
k_dgvol3(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ G, long long nel, Basis1D bs) {
  constexpr int Q = P + 1, Q2 = Q * Q, Q3 = Q * Q * Q;
  __shared__ double sB[Q2], sD[Q2];
  __shared__ double S[EB][3][Q3];
  const int tx = threadIdx.x, ty = threadIdx.y, te = threadIdx.z;
  const int lt = tx + Q * (ty + Q * te);
  for (int i = lt; i < Q2; i += Q2 * EB) { sB[i] = bs.B[i]; sD[i] = bs.D[i]; }
  const long long e = (long long)blockIdx.x * EB + te;
  const bool active = e < nel;
  const double* xe = x + (active ? e : 0) * Q3;
  double u[Q];
#pragma unroll
  for (int c = 0; c < Q; ++c) u[c] = active ? xe[tx + Q * (ty + Q * c)] : 0.0;
  __syncthreads();
  double* S0 = S[te][0];
  double* S1 = S[te][1];
  double* S2 = S[te][2];
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double bu = 0.0, du = 0.0;
#pragma unroll
    for (int c = 0; c < Q; ++c) { bu += sB[qz * Q + c] * u[c]; du += sD[qz * Q + c] * u[c]; }
    S0[qz * Q2 + ty * Q + tx] = bu;
    S1[qz * Q2 + ty * Q + tx] = du;
  }
  __syncthreads();
  double r1[Q], r2[Q], r3[Q];
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
    for (int b = 0; b < Q; ++b) {
      const double s0 = S0[qz * Q2 + b * Q + tx], s1 = S1[qz * Q2 + b * Q + tx];
      t1 += sB[ty * Q + b] * s0; t2 += sD[ty * Q + b] * s0; t3 += sB[ty * Q + b] * s1;
    }
    r1[qz] = t1; r2[qz] = t2; r3[qz] = t3;
  }
  __syncthreads();
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    S0[qz * Q2 + ty * Q + tx] = r1[qz]; S1[qz * Q2 + ty * Q + tx] = r2[qz]; S2[qz * Q2 + ty * Q + tx] = r3[qz];
  }
  __syncthreads();
  const double* Ge = G + (active ? e : 0) * 6 * Q3;
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double gxv = 0.0, gyv = 0.0, gzv = 0.0;
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      gxv += sD[tx * Q + a] * S0[qz * Q2 + ty * Q + a];
      gyv += sB[tx * Q + a] * S1[qz * Q2 + ty * Q + a];
      gzv += sB[tx * Q + a] * S2[qz * Q2 + ty * Q + a];
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
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double w1 = 0.0, w2 = 0.0, w3 = 0.0;
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      w1 += sD[qx * Q + tx] * S0[qz * Q2 + ty * Q + qx];
      w2 += sB[qx * Q + tx] * S1[qz * Q2 + ty * Q + qx];
      w3 += sB[qx * Q + tx] * S2[qz * Q2 + ty * Q + qx];
    }
    r1[qz] = w1; r2[qz] = w2; r3[qz] = w3;
  }
  __syncthreads();
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    S0[qz * Q2 + ty * Q + tx] = r1[qz]; S1[qz * Q2 + ty * Q + tx] = r2[qz]; S2[qz * Q2 + ty * Q + tx] = r3[qz];
  }
  __syncthreads();
  double yb[Q], yd[Q];
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      t1 += sB[qy * Q + ty] * S0[qz * Q2 + qy * Q + tx] + sD[qy * Q + ty] * S1[qz * Q2 + qy * Q + tx];
      t2 += sB[qy * Q + ty] * S2[qz * Q2 + qy * Q + tx];
    }
    yb[qz] = t1; yd[qz] = t2;
  }
  if (!active) return;
  double* ye = y + e * Q3;
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    double v = 0.0;
#pragma unroll
    for (int qz = 0; qz < Q; ++qz) v += sB[qz * Q + c] * yb[qz] + sD[qz * Q + c] * yd[qz];
    ye[tx + Q * (ty + Q * c)] = v;
  }
}

// ----------------------------------------------------------------- face helpers
// axes of a face normal to axis k: tangential t1 < t2
__device__ __forceinline__ void face_axes(int k, int& t1, int& t2) {
  t1 = k == 0 ? 1 : 0;
  t2 = k == 2 ? 1 : 2;
}
// local (element) node index of (a_k, a_t1, a_t2)
template <int Q>
__device__ __forceinline__ int lnode(int k, int t1, int t2, int ak, int i, int j) {
  int a[3];
  a[k] = ak; a[t1] = i; a[t2] = j;
  return a[0] + Q * (a[1] + Q * a[2]);
}
__device__ __forceinline__ long long elem_id(const int* ec, int3 n) {
  return ec[0] + (long long)n.x * (ec[1] + (long long)n.y * ec[2]);
}

struct FaceGeo {
  double Ji[9];
  double det;
};
__device__ __forceinline__ void face_geo(const double* V, int3 n, const int* ec, int k, int side, double xt1, double xt2,
                                         int t1, int t2, FaceGeo& g, double* xp) {
  double xi[3], J[9];
  xi[k] = side ? 1.0 : 0.0;
  xi[t1] = xt1;
  xi[t2] = xt2;
  const int nv[3] = {n.x + 1, n.y + 1, n.z + 1};
  double xx[3];
  elem_map<3>(V, nv, ec[0], ec[1], ec[2], xi, xx, J);
  g.det = inv_det<3>(J, g.Ji);
  if (xp) { xp[0] = xx[0]; xp[1] = xx[1]; xp[2] = xx[2]; }
}

__device__ __forceinline__ double block_sum_small(double v, double* red) {
  // blockDim.x <= 64
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  if (t == 0) {
    double s = 0.0;
    for (int i = 0; i < blockDim.x; ++i) s += red[i];
    red[64] = s;
  }
  __syncthreads();
  const double r = red[64];
  __syncthreads();
  return r;
}

// mode 0: operator face terms for all faces normal to `axis`
// mode 1: boundary RHS (sigma g v - g d_n v) for boundary faces normal to axis on side `bside`
template <int P>
__global__ void __launch_bounds__((P + 1) * (P + 1))
k_dgface3(int mode, int axis, int bside, const double* __restrict__ x, double* __restrict__ y,
          const double* __restrict__ gq, const double* __restrict__ V, const double* __restrict__ vol, int3 n,
          Basis1D bs, double eta, int br2) {
  constexpr int Q = P + 1, Q2 = Q * Q, NL = Q * Q * Q;
  __shared__ double su[2][NL];
  __shared__ double T0[2][Q2], T1[2][Q2];
  __shared__ double X0[2][Q2], X1[2][Q2], X2[2][Q2];
  __shared__ double red[65];
  const int k = axis;
  int t1, t2;
  face_axes(k, t1, t2);
  const int nn[3] = {n.x, n.y, n.z};
  const int tid = threadIdx.x;
  const int qi = tid % Q, qj = tid / Q;
  // decode the face and its elements
  int ecm[3], ecp[3];
  bool hm, hp;
  if (mode == 0) {
    const long long f = blockIdx.x;
    const int fk = (int)(f % (nn[k] + 1));
    const long long rest = f / (nn[k] + 1);
    const int c1 = (int)(rest % nn[t1]), c2 = (int)(rest / nn[t1]);
    ecm[k] = fk - 1; ecm[t1] = c1; ecm[t2] = c2;
    ecp[k] = fk; ecp[t1] = c1; ecp[t2] = c2;
    hm = fk >= 1;
    hp = fk <= nn[k] - 1;
  } else {
    const long long f = blockIdx.x;
    const int c1 = (int)(f % nn[t1]), c2 = (int)(f / nn[t1]);
    ecm[k] = nn[k] - 1; ecm[t1] = c1; ecm[t2] = c2;
    ecp[k] = 0; ecp[t1] = c1; ecp[t2] = c2;
    hm = bside == 1;
    hp = bside == 0;
  }
  const long long em = hm ? elem_id(ecm, n) : -1, ep = hp ? elem_id(ecp, n) : -1;
  // side 0 = K^- (face at xi_k = 1), side 1 = K^+ (face at xi_k = 0)
  const int endn[2] = {P, 0};
  const double* Eend[2] = {bs.E1, bs.E0};
  double u[2] = {0, 0}, g[2][3] = {{0, 0, 0}, {0, 0, 0}};
  if (mode == 0) {
    for (int s = 0; s < 2; ++s) {
      const long long e = s == 0 ? em : ep;
      if (e < 0) continue;
      for (int idx = tid; idx < NL; idx += Q2) su[s][idx] = x[e * NL + idx];
    }
    __syncthreads();
    // slabs: trace (a_k = end) and reference normal derivative sum_a l_a'(end) u
    for (int s = 0; s < 2; ++s) {
      const long long e = s == 0 ? em : ep;
      if (e < 0) continue;
      const int i = qi, j = qj;  // here (i, j) index tangential nodes
      T0[s][i + Q * j] = su[s][lnode<Q>(k, t1, t2, endn[s], i, j)];
      double a = 0.0;
      for (int ak = 0; ak < Q; ++ak) a += Eend[s][ak] * su[s][lnode<Q>(k, t1, t2, ak, i, j)];
      T1[s][i + Q * j] = a;
    }
    __syncthreads();
    // interpolate along t1: thread (qi, j)
    for (int s = 0; s < 2; ++s) {
      const long long e = s == 0 ? em : ep;
      if (e < 0) continue;
      const int j = qj;
      double a0 = 0, a1 = 0, a2 = 0;
      for (int i = 0; i < Q; ++i) {
        a0 += bs.B[qi * Q + i] * T0[s][i + Q * j];
        a1 += bs.D[qi * Q + i] * T0[s][i + Q * j];
        a2 += bs.B[qi * Q + i] * T1[s][i + Q * j];
      }
      X0[s][qi + Q * j] = a0; X1[s][qi + Q * j] = a1; X2[s][qi + Q * j] = a2;
    }
    __syncthreads();
    // along t2: thread (qi, qj) -> u, reference gradient
    for (int s = 0; s < 2; ++s) {
      const long long e = s == 0 ? em : ep;
      if (e < 0) continue;
      double uu = 0, d1 = 0, d2 = 0, dn = 0;
      for (int j = 0; j < Q; ++j) {
        const double bj = bs.B[qj * Q + j];
        uu += bj * X0[s][qi + Q * j];
        d1 += bj * X1[s][qi + Q * j];
        d2 += bs.D[qj * Q + j] * X0[s][qi + Q * j];
        dn += bj * X2[s][qi + Q * j];
      }
      u[s] = uu;
      g[s][k] = dn; g[s][t1] = d1; g[s][t2] = d2;
    }
  }
  // geometry at this face point for each side
  FaceGeo G[2];
  const double w = bs.wq[qi] * bs.wq[qj];
  const int sref = hm ? 0 : 1;  // side whose outward normal defines n (K^- if present)
  for (int s = 0; s < 2; ++s) {
    const long long e = s == 0 ? em : ep;
    if (e < 0) continue;
    face_geo(V, n, s == 0 ? ecm : ecp, k, s == 0 ? 1 : 0, bs.xq[qi], bs.xq[qj], t1, t2, G[s], nullptr);
  }
  double nr = 0.0;
  for (int m = 0; m < 3; ++m) nr += G[sref].Ji[k * 3 + m] * G[sref].Ji[k * 3 + m];
  nr = sqrt(nr);
  double nv[3];
  const double sg = sref == 0 ? 1.0 : -1.0;
  for (int m = 0; m < 3; ++m) nv[m] = sg * G[sref].Ji[k * 3 + m] / nr;
  const double dS = w * G[sref].det * nr;
  const double area = block_sum_small(dS, red);
  double hv;
  if (hm && hp) hv = fmin(vol[em], vol[ep]);
  else hv = vol[hm ? em : ep];
  const double sigma = eta / (hv / area);
  // the jump J at this point ([u] = J n): interior u^- - u^+, boundary u (or the data g)
  double Jq = 0.0;
  if (mode == 0) Jq = (hm && hp) ? u[0] - u[1] : u[sref];
  else Jq = gq[(long long)blockIdx.x * Q2 + tid];
  // BR2 (eq:br2, lifting eq:lift): the penalty value sigma J is replaced by
  //   g = eta sum_K s_K^2 sum_m n_m W_m^K,  W_m^K = sum_i (M_K^{-1} b_m^K)_i psi_i^K,
  //   b_m^K,i = int_e J n_m psi_i^K.
  // Affine elements: M_K = det J_K (M1 x M1 x M1), only face nodes of K see the face,
  // so M_K^{-1} on them is (M1^{-1})_{end,end} (M1^{-1} x M1^{-1}) / det J_K and the two
  // sides share b (same tangential basis); flat faces: sum_m n_m n_m = 1.
  double pen = sigma * Jq;
  if (br2) {
    X0[0][tid] = dS * Jq;
    __syncthreads();
    {  // beta[i][j] = sum_q B[q1][i] B[q2][j] dS J   (transpose interpolation)
      double a = 0.0;
      for (int q1 = 0; q1 < Q; ++q1) a += bs.B[q1 * Q + qi] * X0[0][q1 + Q * qj];
      X1[0][qi + Q * qj] = a;
    }
    __syncthreads();
    {
      double a = 0.0;
      for (int q2 = 0; q2 < Q; ++q2) a += bs.B[q2 * Q + qj] * X1[0][qi + Q * q2];
      X2[0][tid] = a;  // beta[qi][qj]
    }
    __syncthreads();
    {  // c = (M1^{-1} x M1^{-1}) beta
      double a = 0.0;
      for (int i2 = 0; i2 < Q; ++i2) a += bs.M1inv[qi * Q + i2] * X2[0][i2 + Q * qj];
      X0[1][tid] = a;
    }
    __syncthreads();
    {
      double a = 0.0;
      for (int j2 = 0; j2 < Q; ++j2) a += bs.M1inv[qj * Q + j2] * X0[1][qi + Q * j2];
      X1[1][tid] = a;  // c[qi][qj]
    }
    __syncthreads();
    {  // W at the point (q1 = qi, q2 = qj)
      double a = 0.0;
      for (int i = 0; i < Q; ++i) a += bs.B[qi * Q + i] * X1[1][i + Q * qj];
      X2[1][qi + Q * qj] = a;
    }
    __syncthreads();
    double W = 0.0;
    for (int j = 0; j < Q; ++j) W += bs.B[qj * Q + j] * X2[1][qi + Q * j];
    const double kap = bs.M1inv[0];
    double coef;
    if (hm && hp) coef = 0.25 * kap * (1.0 / G[0].det + 1.0 / G[1].det);
    else coef = kap / G[sref].det;
    pen = eta * coef * W;
    __syncthreads();
  }
  // point coefficients: c_phi (value test) and c_g (normal-derivative test, along n)
  double cphi[2] = {0, 0}, cg[2] = {0, 0};
  if (mode == 0) {
    double dnu[2] = {0, 0};
    for (int s = 0; s < 2; ++s) {
      const long long e = s == 0 ? em : ep;
      if (e < 0) continue;
      double a = 0.0;
      for (int m = 0; m < 3; ++m) {
        double gm = 0.0;
        for (int r = 0; r < 3; ++r) gm += G[s].Ji[r * 3 + m] * g[s][r];
        a += gm * nv[m];
      }
      dnu[s] = a;
    }
    if (hm && hp) {
      const double avg = 0.5 * (dnu[0] + dnu[1]);
      cphi[0] = dS * (-avg + pen); cg[0] = -0.5 * dS * Jq;
      cphi[1] = dS * (avg - pen);  cg[1] = -0.5 * dS * Jq;
    } else {
      const int s = sref;
      cphi[s] = dS * (-dnu[s] + pen);
      cg[s] = -dS * Jq;
    }
  } else {
    // boundary data g at this point: ordering (axis, side, elements ascending, points)
    cphi[sref] = dS * pen;
    cg[sref] = -dS * Jq;
  }
  // transpose: reference-direction weights of the gradient test term
  for (int s = 0; s < 2; ++s) {
    const long long e = s == 0 ? em : ep;
    if (e < 0) continue;
    double wr[3];
    for (int r = 0; r < 3; ++r) {
      double a = 0.0;
      for (int m = 0; m < 3; ++m) a += G[s].Ji[r * 3 + m] * nv[m];
      wr[r] = cg[s] * a;
    }
    // point arrays [qi + Q qj]
    X0[s][tid] = cphi[s];
    X1[s][tid] = wr[t1];
    X2[s][tid] = wr[t2];
    T1[s][tid] = wr[k];
  }
  __syncthreads();
  // along t2 (transpose): thread (qi, j)
  double y0[2] = {0, 0}, y1[2] = {0, 0}, y2[2] = {0, 0};
  for (int s = 0; s < 2; ++s) {
    const long long e = s == 0 ? em : ep;
    if (e < 0) continue;
    const int j = qj;
    double a0 = 0, a1 = 0, a2 = 0;
    for (int q2 = 0; q2 < Q; ++q2) {
      const double b = bs.B[q2 * Q + j];
      a0 += b * X0[s][qi + Q * q2] + bs.D[q2 * Q + j] * X2[s][qi + Q * q2];
      a1 += b * X1[s][qi + Q * q2];
      a2 += b * T1[s][qi + Q * q2];
    }
    y0[s] = a0; y1[s] = a1; y2[s] = a2;
  }
  __syncthreads();
  for (int s = 0; s < 2; ++s) {
    if ((s == 0 ? em : ep) < 0) continue;
    X0[s][tid] = y0[s]; X1[s][tid] = y1[s]; X2[s][tid] = y2[s];   // indexed [qi + Q j]
  }
  __syncthreads();
  // along t1 (transpose): thread (i, j) -> trace slab S0 and normal slab S1
  for (int s = 0; s < 2; ++s) {
    const long long e = s == 0 ? em : ep;
    if (e < 0) continue;
    const int i = qi, j = qj;
    double s0 = 0.0, s1 = 0.0;
    for (int q1 = 0; q1 < Q; ++q1) {
      s0 += bs.B[q1 * Q + i] * X0[s][q1 + Q * j] + bs.D[q1 * Q + i] * X1[s][q1 + Q * j];
      s1 += bs.B[q1 * Q + i] * X2[s][q1 + Q * j];
    }
    double* ye = y + e * NL;
    for (int ak = 0; ak < Q; ++ak) {
      double v = Eend[s][ak] * s1;
      if (ak == endn[s]) v += s0;
      atomicAdd(ye + lnode<Q>(k, t1, t2, ak, i, j), v);
    }
  }
}

// boundary-face Gauss point coordinates (ordering: axis, side, elements, points)
__global__ void k_bface_points(double* __restrict__ X, const double* __restrict__ V, int3 n, Basis1D bs, int axis,
                               int bside, long long base) {
  const int Q = bs.q;
  const int tid = threadIdx.x;
  if (tid >= Q * Q) return;
  const int qi = tid % Q, qj = tid / Q;
  int t1, t2;
  face_axes(axis, t1, t2);
  const int nn[3] = {n.x, n.y, n.z};
  const long long f = blockIdx.x;
  int ec[3];
  ec[axis] = bside ? nn[axis] - 1 : 0;
  ec[t1] = (int)(f % nn[t1]);
  ec[t2] = (int)(f / nn[t1]);
  FaceGeo G;
  double xp[3];
  face_geo(V, n, ec, axis, bside, bs.xq[qi], bs.xq[qj], t1, t2, G, xp);
  const long long o = base + f * Q * Q + tid;
  for (int m = 0; m < 3; ++m) X[o * 3 + m] = xp[m];
}

// diag(A_IP): volume |grad phi_a|^2 + faces (sigma phi^2 - c phi d_n phi), c = 1
// interior, 2 boundary (written out from eq:ip; thread per DG dof; setup only)
__global__ void k_dgdiag3(double* __restrict__ Dg, const double* __restrict__ V, const double* __restrict__ vol, int3 n,
                          Basis1D bs, double eta, int br2) {
  const int p = bs.p, Q = bs.q, NL = Q * Q * Q;
  const long long nel = (long long)n.x * n.y * n.z;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nel * NL) return;
  const long long e = t / NL;
  const int a = (int)(t % NL);
  const int ac[3] = {a % Q, (a / Q) % Q, a / (Q * Q)};
  const int ec[3] = {(int)(e % n.x), (int)((e / n.x) % n.y), (int)(e / ((long long)n.x * n.y))};
  const int nn[3] = {n.x, n.y, n.z};
  const int nv[3] = {n.x + 1, n.y + 1, n.z + 1};
  double acc = 0.0;
  for (int iq = 0; iq < Q * Q * Q; ++iq) {
    const int qc[3] = {iq % Q, (iq / Q) % Q, iq / (Q * Q)};
    double xi[3], xx[3], J[9], Ji[9], w = 1.0, gr[3];
    for (int m = 0; m < 3; ++m) { xi[m] = bs.xq[qc[m]]; w *= bs.wq[qc[m]]; }
    elem_map<3>(V, nv, ec[0], ec[1], ec[2], xi, xx, J);
    const double det = inv_det<3>(J, Ji);
    for (int r = 0; r < 3; ++r) {
      double gg = 1.0;
      for (int m = 0; m < 3; ++m) gg *= (m == r ? bs.D : bs.B)[qc[m] * Q + ac[m]];
      gr[r] = gg;
    }
    double s = 0.0;
    for (int m = 0; m < 3; ++m) {
      double gm = 0.0;
      for (int r = 0; r < 3; ++r) gm += Ji[r * 3 + m] * gr[r];
      s += gm * gm;
    }
    acc += w * det * s;
  }
  for (int k = 0; k < 3; ++k)
    for (int side = 0; side < 2; ++side) {
      if (ac[k] != (side ? p : 0)) continue;  // phi_a vanishes on this face
      int t1, t2;
      face_axes(k, t1, t2);
      int nb[3] = {ec[0], ec[1], ec[2]};
      nb[k] += side ? 1 : -1;
      const bool interior = nb[k] >= 0 && nb[k] < nn[k];
      const double* E = side ? bs.E1 : bs.E0;
      const double sg = side ? 1.0 : -1.0;
      double area = 0.0, s_pp = 0.0, s_pd = 0.0, det_me = 1.0;
      double beta[(MAXP + 1) * (MAXP + 1)];   // BR2: int_e phi_a psi_(i,j) dS on the face nodes
      for (int i = 0; i < Q * Q; ++i) beta[i] = 0.0;
      for (int qj = 0; qj < Q; ++qj)
        for (int qi = 0; qi < Q; ++qi) {
          FaceGeo G;
          face_geo(V, n, ec, k, side, bs.xq[qi], bs.xq[qj], t1, t2, G, nullptr);
          det_me = G.det;
          double nr = 0.0;
          for (int m = 0; m < 3; ++m) nr += G.Ji[k * 3 + m] * G.Ji[k * 3 + m];
          nr = sqrt(nr);
          const double dS = bs.wq[qi] * bs.wq[qj] * G.det * nr;
          const double phi = bs.B[qi * Q + ac[t1]] * bs.B[qj * Q + ac[t2]];
          double gr[3];
          gr[k] = E[ac[k]] * phi;
          gr[t1] = bs.D[qi * Q + ac[t1]] * bs.B[qj * Q + ac[t2]];
          gr[t2] = bs.B[qi * Q + ac[t1]] * bs.D[qj * Q + ac[t2]];
          double dn = 0.0;
          for (int m = 0; m < 3; ++m) {
            double gm = 0.0;
            for (int r = 0; r < 3; ++r) gm += G.Ji[r * 3 + m] * gr[r];
            dn += gm * sg * G.Ji[k * 3 + m] / nr;
          }
          area += dS;
          s_pp += dS * phi * phi;
          s_pd += dS * phi * dn;
          if (br2)
            for (int j = 0; j < Q; ++j)
              for (int i = 0; i < Q; ++i) beta[i + Q * j] += dS * phi * bs.B[qi * Q + i] * bs.B[qj * Q + j];
        }
      const double hv = interior ? fmin(vol[e], vol[elem_id(nb, n)]) : vol[e];
      double pen;
      if (!br2) {
        pen = eta / (hv / area) * s_pp;
      } else {
        // eta sum_K s_K^2 b(phi_a)^T M_K^{-1} b(phi_a), affine M_K (see k_dgface3)
        double quad = 0.0;
        for (int j = 0; j < Q; ++j)
          for (int i = 0; i < Q; ++i) {
            double c = 0.0;
            for (int j2 = 0; j2 < Q; ++j2)
              for (int i2 = 0; i2 < Q; ++i2) c += bs.M1inv[i * Q + i2] * bs.M1inv[j * Q + j2] * beta[i2 + Q * j2];
            quad += beta[i + Q * j] * c;
          }
        double inv_det = 1.0 / det_me;
        double s2 = 1.0;
        if (interior) {
          FaceGeo Gn;
          face_geo(V, n, nb, k, side ? 0 : 1, bs.xq[0], bs.xq[0], t1, t2, Gn, nullptr);
          inv_det += 1.0 / Gn.det;
          s2 = 0.25;
        }
        pen = eta * s2 * bs.M1inv[0] * inv_det * quad;
      }
      acc += pen - (interior ? 1.0 : 2.0) * s_pd;
    }
  Dg[t] = acc;
}

// r_cg = E^T r_dg on free CG nodes (sum over the DG copies of each node, fixed order)
__global__ void k_dg_restrict(const double* __restrict__ rdg, double* __restrict__ rcg, int3 n, int3 N, int p) {
  const long long NT = (long long)N.x * N.y * N.z;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= NT) return;
  const int gc[3] = {(int)(g % N.x), (int)((g / N.x) % N.y), (int)(g / ((long long)N.x * N.y))};
  const int Nn[3] = {N.x, N.y, N.z}, nn[3] = {n.x, n.y, n.z};
  bool dir = false;
  for (int k = 0; k < 3; ++k) if (gc[k] == 0 || gc[k] == Nn[k] - 1) dir = true;
  if (dir) { rcg[g] = 0.0; return; }
  const int Q = p + 1;
  int lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = max((gc[k] - 1) / p, 0);
    hi[k] = min(gc[k] / p, nn[k] - 1);
  }
  double s = 0.0;
  for (int ez = lo[2]; ez <= hi[2]; ++ez)
    for (int ey = lo[1]; ey <= hi[1]; ++ey)
      for (int ex = lo[0]; ex <= hi[0]; ++ex) {
        const int a0 = gc[0] - ex * p, a1 = gc[1] - ey * p, a2 = gc[2] - ez * p;
        if (a0 < 0 || a0 > p || a1 < 0 || a1 > p || a2 < 0 || a2 > p) continue;
        const long long e = ex + (long long)n.x * (ey + (long long)n.y * ez);
        s += rdg[e * Q * Q * Q + a0 + Q * (a1 + Q * a2)];
      }
  rcg[g] = s;
}

// z_dg = E z_cg + S_B D_B^{-1} S_B^T r_dg (eq:dg-as; point Jacobi on V_B, reading c16)
__global__ void k_dg_combine(const double* __restrict__ rdg, const double* __restrict__ zcg, const double* __restrict__ Dg,
                             double* __restrict__ zdg, int3 n, int3 N, int p) {
  const int Q = p + 1, NL = Q * Q * Q;
  const long long nel = (long long)n.x * n.y * n.z;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nel * NL) return;
  const long long e = t / NL;
  const int a = (int)(t % NL);
  const int ac[3] = {a % Q, (a / Q) % Q, a / (Q * Q)};
  const int ec[3] = {(int)(e % n.x), (int)((e / n.x) % n.y), (int)(e / ((long long)n.x * n.y))};
  const long long g = (ec[0] * p + ac[0]) + (long long)N.x * ((ec[1] * p + ac[1]) + (long long)N.y * (ec[2] * p + ac[2]));
  double v = zcg[g];
  bool bnd = false;
  for (int k = 0; k < 3; ++k) if (ac[k] == 0 || ac[k] == p) bnd = true;
  if (bnd) v += rdg[t] / Dg[t];
  zdg[t] = v;
}

template <int P>
static void launch_faces(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s) {
  constexpr int Q = P + 1;
  const int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  for (int k = 0; k < 3; ++k) {
    long long nf = (long long)(m->n[k] + 1) * (m->nel / m->n[k]);
    k_dgface3<P><<<(unsigned)nf, Q * Q, 0, s>>>(0, k, 0, x, y, nullptr, m->V, m->vol, n, m->basis, m->desc.eta,
                                                 m->desc.disc == 2);
  }
}
template <int P, int EB>
static void launch_vol(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s) {
  constexpr int Q = P + 1;
  dim3 blk(Q, Q, EB);
  k_dgvol3<P, EB><<<(unsigned)((m->nel + EB - 1) / EB), blk, 0, s>>>(x, y, m->G, m->nel, m->basis);
}

int dg_apply(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s) {
  if (m->d != 3) return fail(LORPC_ERR_SIZE, "dg: 3D only");
  switch (m->p) {
    case 1: launch_vol<1, 8>(m, x, y, s); break;
    case 2: launch_vol<2, 8>(m, x, y, s); break;
    case 3: launch_vol<3, 8>(m, x, y, s); break;
    case 4: launch_vol<4, 4>(m, x, y, s); break;
    case 5: launch_vol<5, 4>(m, x, y, s); break;
    case 6: launch_vol<6, 2>(m, x, y, s); break;
    default: return fail(LORPC_ERR_SIZE, "dg: p not compiled");
  }
  LORPC_LAUNCHED();
  switch (m->p) {
    case 1: launch_faces<1>(m, x, y, s); break;
    case 2: launch_faces<2>(m, x, y, s); break;
    case 3: launch_faces<3>(m, x, y, s); break;
    case 4: launch_faces<4>(m, x, y, s); break;
    case 5: launch_faces<5>(m, x, y, s); break;
    case 6: launch_faces<6>(m, x, y, s); break;
  }
  for (int k = 0; k < 3; ++k) LORPC_LAUNCHED();
  return LORPC_OK;
}

int dg_diag_setup(lorpc_mesh* m, cudaStream_t s) {
  if (m->d != 3) return fail(LORPC_ERR_SIZE, "dg: 3D only");
  LORPC_TRY(dalloc(&m->dgdiag, (size_t)m->ndof));
  const int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  k_dgdiag3<<<(unsigned)((m->ndof + 127) / 128), 128, 0, s>>>(m->dgdiag, m->V, m->vol, n, m->basis, m->desc.eta,
                                                              m->desc.disc == 2);
  LORPC_LAUNCHED();
  std::vector<double> h(m->ndof);
  LORPC_CUDA(cudaMemcpyAsync(h.data(), m->dgdiag, sizeof(double) * m->ndof, cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  for (long long i = 0; i < m->ndof; ++i)
    if (!(h[i] > 0.0)) return fail(LORPC_ERR_ARG, "dg: non-positive diagonal at dof " + std::to_string(i));
  return LORPC_OK;
}

int dg_restrict_cg(const lorpc_mesh* m, const double* r_dg, double* r_cg, cudaStream_t s) {
  const int3 n = make_int3(m->n[0], m->n[1], m->n[2]), N = make_int3(m->N[0], m->N[1], m->N[2]);
  k_dg_restrict<<<(unsigned)((m->ndof_cg + 255) / 256), 256, 0, s>>>(r_dg, r_cg, n, N, m->p);
  LORPC_LAUNCHED();
  return LORPC_OK;
}

int dg_combine(const lorpc_mesh* m, const double* r_dg, const double* z_cg, double* z_dg, cudaStream_t s) {
  const int3 n = make_int3(m->n[0], m->n[1], m->n[2]), N = make_int3(m->N[0], m->N[1], m->N[2]);
  k_dg_combine<<<(unsigned)((m->ndof + 255) / 256), 256, 0, s>>>(r_dg, z_cg, m->dgdiag, z_dg, n, N, m->p);
  LORPC_LAUNCHED();
  return LORPC_OK;
}

int dg_bface_points(const lorpc_mesh* m, double* xbq, cudaStream_t s) {
  if (m->d != 3) return fail(LORPC_ERR_SIZE, "dg: 3D only");
  const int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  const int Q2 = m->q * m->q;
  long long base = 0;
  for (int k = 0; k < 3; ++k)
    for (int side = 0; side < 2; ++side) {
      const long long nf = m->nel / m->n[k];
      k_bface_points<<<(unsigned)nf, Q2, 0, s>>>(xbq, m->V, n, m->basis, k, side, base);
      LORPC_LAUNCHED();
      base += nf * Q2;
    }
  return LORPC_OK;
}

template <int P>
static void launch_bc(const lorpc_mesh* m, const double* gq, double* b, cudaStream_t s) {
  constexpr int Q = P + 1;
  const int3 n = make_int3(m->n[0], m->n[1], m->n[2]);
  long long base = 0;
  for (int k = 0; k < 3; ++k)
    for (int side = 0; side < 2; ++side) {
      const long long nf = m->nel / m->n[k];
      k_dgface3<P><<<(unsigned)nf, Q * Q, 0, s>>>(1, k, side, nullptr, b, gq + base, m->V, m->vol, n, m->basis,
                                                 m->desc.eta, m->desc.disc == 2);
      base += nf * Q * Q;
    }
}

int dg_rhs_bc(const lorpc_mesh* m, const double* gq, double* b, cudaStream_t s) {
  switch (m->p) {
    case 1: launch_bc<1>(m, gq, b, s); break;
    case 2: launch_bc<2>(m, gq, b, s); break;
    case 3: launch_bc<3>(m, gq, b, s); break;
    case 4: launch_bc<4>(m, gq, b, s); break;
    case 5: launch_bc<5>(m, gq, b, s); break;
    case 6: launch_bc<6>(m, gq, b, s); break;
    default: return fail(LORPC_ERR_SIZE, "dg: p not compiled");
  }
  for (int i = 0; i < 6; ++i) LORPC_LAUNCHED();
  return LORPC_OK;
}

}  // namespace lorpc
