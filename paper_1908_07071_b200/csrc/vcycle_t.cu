// Thread-per-patch Schwarz V-cycle (rows a5, a6, a8; "patches are
// processed independently and batched").
//
// One lane owns one patch, one warp owns 32 patches.  The MDF-ordered ILU(0)
// sweeps, a strictly sequential chain per patch, run lane-parallel over the warp's
// 32 patches with no synchronisation and no reductions: lane q walks its own
// patch's rows in its DAG-schedule order.  The factors are stored warp-interleaved
// ("T-records", built from the per-patch records at setup) so that every load of a
// sweep step is one coalesced row; a step is padded to the warp's widest column
// and the padding lanes are predicated off (no memory traffic).
//
// Three kernels per apply: pre-smoothing (gather r_j = I_j^T r, x = M^{-1} r_j),
// the coarse correction (lane = patch: s = r_j - A x, r_1 = P^T s, z_1 = C r_1
// with C the dense V-cycle operator of levels >= 1, y = x + P z_1, s = r_j - A y)
// and post-smoothing (z_j = y + M^{-1} s, scatter z += I_j z_j).  The patch
// vectors travel between them in warp-interleaved "park" buffers [warp][node][32].
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "patch.cuh"

namespace lorpc {

// ------------------------------------------------------------------ warp slots
// Warp w owns the patches pord[32 w .. 32 w + 31] (-1: empty slot, only in the
// last warp).  The patch grid is walked in tiles of TX x TY patch columns, each
// tile bottom to top (z outer), so that patches sharing LOR rows and r / z entries
// run at nearly the same time and meet in L2: z-neighbours are one tile layer
// (TX * TY patches) apart, while lexicographic order puts them a whole patch plane
// apart, beyond the L2 reuse window of the concurrently resident warps.
std::vector<int> tile_order(const lorpc_prec* b, int TX, int TY) {
  const lorpc_mesh* m = b->m;
  const int d = m->d, star = b->desc.patch_kind == 1;
  const int gx = m->n[0] + (star ? 0 : 1), gy = m->n[1] + (star ? 0 : 1);
  const int gz = d == 3 ? (star ? m->n[2] : b->pnvz) : 1;
  const long long nw = (b->J + 31) / 32;
  std::vector<int> ord;
  ord.reserve((size_t)(nw * 32));
  for (int y0 = 0; y0 < gy; y0 += TY)
    for (int x0 = 0; x0 < gx; x0 += TX)
      for (int z = 0; z < gz; ++z)
        for (int y = y0; y < std::min(y0 + TY, gy); ++y)
          for (int x = x0; x < std::min(x0 + TX, gx); ++x) ord.push_back(x + gx * (y + gy * z));
  ord.resize((size_t)(nw * 32), -1);
  return ord;
}

// ------------------------------------------------------------------ T-records
// Block of (warp w, level 0) at trecoff[w], 256-byte aligned.  Step t of lane q
// stores the COLUMN of its node k: the entries L_ik of the later neighbours i.  The
// forward sweep pushes (y_i -= L_ik y_k, then x_k = y_k / D_k) and the backward
// sweep pulls (x_k -= sum_i L_ik x_i, steps descending) from the same data, so the
// factor is stored once and the backward sweep re-reads, in reverse, what the
// forward sweep has just pulled through L2:
//   int4 {S, Kp, 0, 0}: S steps (largest patch of the warp), Kp pair rows
//   hdr[S][32]  u32  node k (bits 0-15) | count (bits 16-23) | mp (bits 24-31): pair
//                    rows of step t (the warp maximum, the same in every lane)
//   Dinv[S][32] f64  1 / D_k
//   Lc[Kp][32]  f64x2 column entries in pairs (one 16-byte load per lane and pair)
//   Ic[Kp][32]  their node indices i: u8x2 when the largest patch has <= 254 nodes
//               (tiw = 1: C5, C2), else u16x2 (tiw = 2: C3)
// Padding entries carry L = 0 and the dummy node n0max, padding steps the dummy
// node with count 0.
struct TRecLayout { long long hdr, D, Lc, Ic, total; };
// node index width of a warp's records: 1 byte when the largest patch has <= 254
// nodes (C5, C2), else 2 bytes (C3)
__host__ __device__ __forceinline__ int tiw(int n0max) { return n0max <= 254 ? 1 : 2; }
__host__ __device__ __forceinline__ long long a256(long long b) { return (b + 255) & ~255ll; }
__host__ __device__ __forceinline__ TRecLayout trec_layout(int S, int Kp, int iw) {
  TRecLayout T;
  T.hdr = 256;
  T.D = a256(T.hdr + 128ll * S);
  T.Lc = T.D + 256ll * S;
  T.Ic = T.Lc + 512ll * Kp;
  T.total = a256(T.Ic + 64ll * iw * Kp);
  return T;
}

// Pair rows per step are padded up to a class {0, 1, 2, 4, 7, 10, 13}: the sweeps
// run a compile-time-sized body per class (no per-step dispatch inside a run of
// equal classes; the MDF columns of a patch plateau at 6-7 pairs).
__host__ __device__ __forceinline__ int tclass(int mp) {
  return mp <= 2 ? mp : mp <= 4 ? 4 : mp <= 7 ? 7 : mp <= 10 ? 10 : 13;
}

struct TRecParams {
  const char* rec;
  const long long* recoff;
  const int* pord;
  int L;
  int dummy;
  long long* sizes;
  char* trec;
  const long long* trecoff;
};

// fill = 0: block sizes; fill = 1: write the blocks.  Thread = warp slot.
__global__ void __launch_bounds__(128) k_trec(TRecParams P, long long nslots, int fill) {
  const long long slot = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if ((slot & ~31ll) >= nslots) return;  // warp-uniform
  const long long w = slot >> 5;
  const int lane = threadIdx.x & 31;
  const long long j = P.pord[slot];
  int n = 0, nL = 0;
  const char* rec = P.rec;
  if (j >= 0) {
    rec = P.rec + P.recoff[j * P.L];
    const int4 h = *(const int4*)rec;
    n = h.x; nL = h.z;
  }
  const RecLayout R = rec_layout(n, nL);
  const uint16_t* brp = (const uint16_t*)(rec + R.brp);
  const int S = (int)__reduce_max_sync(0xffffffffu, (unsigned)n);
  int Kp = 0;
  for (int t = 0; t < S; ++t) {
    const unsigned cb = t < n ? brp[t + 1] - brp[t] : 0u;
    Kp += tclass((int)__reduce_max_sync(0xffffffffu, (cb + 1) / 2));
  }
  const int iw = tiw(P.dummy);
  const TRecLayout T = trec_layout(S, Kp, iw);
  if (!fill) {
    if (lane == 0) P.sizes[w] = T.total;
    return;
  }
  char* blk = P.trec + P.trecoff[w];
  if (lane == 0) *(int4*)blk = make_int4(S, Kp, 0, 0);
  uint32_t* H = (uint32_t*)(blk + T.hdr);
  double* Dd = (double*)(blk + T.D);
  double* Lc = (double*)(blk + T.Lc);
  char* Ic = blk + T.Ic;
  const double* Dn = (const double*)(rec + R.D);
  const double* bLv = (const double*)(rec + R.bL);
  const uint16_t* bkv = (const uint16_t*)(rec + R.bk);
  const uint16_t* sch = (const uint16_t*)(rec + R.sched);
  int kp = 0;
  for (int t = 0; t < S; ++t) {
    int node = P.dummy, b0 = 0;
    unsigned cb = 0;
    double dv = 1.0;
    if (t < n) {
      node = sch[t];
      b0 = brp[t]; cb = brp[t + 1] - b0;
      dv = 1.0 / Dn[node];
    }
    const int mp = tclass((int)__reduce_max_sync(0xffffffffu, (cb + 1) / 2));
    H[t * 32 + lane] = (uint32_t)node | (cb << 16) | ((uint32_t)mp << 24);
    Dd[t * 32 + lane] = dv;
    for (int k = 0; k < 2 * mp; ++k) {
      const bool in = k < (int)cb;
      const long long ix = ((long long)(kp + k / 2) * 32 + lane) * 2 + (k & 1);
      Lc[ix] = in ? bLv[b0 + k] : 0.0;
      const int nd = in ? bkv[b0 + k] : P.dummy;
      if (iw == 1) ((uint8_t*)Ic)[ix] = (uint8_t)nd; else ((uint16_t*)Ic)[ix] = (uint16_t)nd;
    }
    kp += mp;
  }
}

// patch geometry: element box and the free-node boxes of levels 0 and 1
struct TPatch { int lo[3], ext[3], cext[3], ec[3], n, n1; };
static_assert(sizeof(TPatch) % sizeof(double) == 0, "TPatch packs into doubles");
template <int DIM>
__device__ __forceinline__ TPatch tpatch(const PatchGeom& G, long long j) {
  TPatch c;
  int elo[3], ehi[3];
  patch_elems(G, j, elo, ehi);
  c.n = c.n1 = 1;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c.ec[k] = ehi[k] - elo[k] + 1;
    if (k >= DIM) { c.lo[k] = 0; c.ext[k] = c.cext[k] = 1; continue; }
    c.lo[k] = elo[k] * (G.ml[0] - 1) + 1;
    c.ext[k] = c.ec[k] * (G.ml[0] - 1) - 1;
    c.cext[k] = c.ec[k] * (G.ml[1] - 1) - 1;
    c.n *= c.ext[k];
    c.n1 *= c.cext[k];
  }
  return c;
}

// Level-1 (coarse) box of the thread kernel: at most CX x CX x CZ nodes.  The dense
// V-cycle operator C of levels >= 1 (symmetric, reading c5) is stored as the upper
// triangle of this fixed box, interleaved by warp slot: Cp[w][idx][32], idx over
// (a <= b) row by row; coarse nodes a clipped boundary patch lacks have zero rows.
template <int DIM> struct TCoarse {
  static constexpr int CX = DIM == 3 ? 3 : 5, CZ = DIM == 3 ? 3 : 1, NC = CX * CX * CZ;
  static constexpr int NPK = NC * (NC + 1) / 2;
};

template <int DIM>
__global__ void k_pack_c(const double* __restrict__ Cd, double* __restrict__ Cp, const int* __restrict__ pord,
                         PatchGeom G, long long nslots, int ldc) {
  constexpr int CX = TCoarse<DIM>::CX, NC = TCoarse<DIM>::NC, NPK = TCoarse<DIM>::NPK;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nslots * NPK) return;
  const int q = (int)(t % 32);
  int idx = (int)((t / 32) % NPK);
  const long long w = t / (32ll * NPK);
  const long long j = pord[w * 32 + q];
  double v = 0.0;
  if (j >= 0) {
    int a = 0;
    while (idx >= NC - a) { idx -= NC - a; ++a; }
    const int bb = a + idx;
    const TPatch c = tpatch<DIM>(G, j);
    const int ax = a % CX, ay = (a / CX) % CX, az = a / (CX * CX);
    const int bx = bb % CX, by = (bb / CX) % CX, bz = bb / (CX * CX);
    if (ax < c.cext[0] && ay < c.cext[1] && az < c.cext[2] && bx < c.cext[0] && by < c.cext[1] && bz < c.cext[2]) {
      const int ia = ax + c.cext[0] * (ay + c.cext[1] * az), ib = bx + c.cext[0] * (by + c.cext[1] * bz);
      v = Cd[j * ldc + (long long)ia * c.n1 + ib];
    }
  }
  Cp[t] = v;
}

// ------------------------------------------------------------------ U-records
// Structure-only orderings (natural, RCM = reading r5) give every patch with the
// same free-node box the same elimination order and the same factor sparsity, so
// the 32 patches of a warp (grouped by box shape) share ONE sweep schedule.  The
// U-record stores that schedule once, as a 32-byte descriptor per step read
// warp-uniformly, and per lane only the factor VALUES: no per-lane node indices or
// headers and no padding to the warp's widest column (T-records), i.e. the L and
// D of the factor plus at most one zero entry per odd column.  P:606-608: "MDF-
// ordered and RCM-ordered ILU give comparable iteration counts".
// Block of warp w at trecoff[w], 256-byte aligned:
//   int4 {S, E2, 0, 0}: S steps, E2 pair rows
//   desc[S]     32 B: node k (byte 0), pair rows mp (byte 1), first pair row kp
//               (bytes 2-3, u16), the 2 mp column nodes i (bytes 4.., u8; the dummy
//               node n0max for the padding entry of an odd column)
//   Dinv[S][32] f64    1 / D_k
//   Lc[E2][32]  f64x2  column entries L_ik in pairs, steps consecutive
struct URecLayout { long long desc, D, Lc, total; };
__host__ __device__ __forceinline__ URecLayout urec_layout(int S, int E2) {
  URecLayout U;
  U.desc = 256;
  U.D = a256(U.desc + 32ll * S);
  U.Lc = U.D + 256ll * S;
  U.total = a256(U.Lc + 512ll * E2);
  return U;
}
constexpr int UMP = 13;  // largest pair count of a column (3D: <= 26 later neighbours)

// One thread per warp slot.  fill = 0: check that the valid lanes of the warp share
// one schedule (node of every step and column nodes; *bad = 1 otherwise) and size
// the block; fill = 1: write it.  Empty slots get zero values (their vectors stay 0).
__global__ void __launch_bounds__(128) k_urec(TRecParams P, long long nslots, int fill, int* bad) {
  const long long slot = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if ((slot & ~31ll) >= nslots) return;  // warp-uniform
  const long long w = slot >> 5;
  const int lane = threadIdx.x & 31;
  const long long j = P.pord[slot];
  int n = 0, nL = 0;
  const char* rec = P.rec;
  if (j >= 0) {
    rec = P.rec + P.recoff[j * P.L];
    const int4 h = *(const int4*)rec;
    n = h.x; nL = h.z;
  }
  const bool valid = j >= 0 && n > 0;
  const unsigned vm = __ballot_sync(0xffffffffu, valid);
  const int ref = vm ? __ffs(vm) - 1 : 0;
  const int S = vm ? __shfl_sync(0xffffffffu, n, ref) : 0;
  const RecLayout R = rec_layout(n, nL);
  const uint16_t* brp = (const uint16_t*)(rec + R.brp);
  const uint16_t* sch = (const uint16_t*)(rec + R.sched);
  const uint16_t* bkv = (const uint16_t*)(rec + R.bk);
  const double* bLv = (const double*)(rec + R.bL);
  const double* Dn = (const double*)(rec + R.D);
  const URecLayout U = urec_layout(S, 0);
  char* blk = fill ? P.trec + P.trecoff[w] : nullptr;
  unsigned char* desc = fill ? (unsigned char*)(blk + U.desc) : nullptr;
  double* Dd = fill ? (double*)(blk + U.D) : nullptr;
  double* Lc = fill ? (double*)(blk + U.Lc) : nullptr;
  bool mism = valid && n != S;
  int kp = 0, mpw = 0;
  for (int t = 0; t < S; ++t) {
    int node = 0, b0 = 0, cb = 0;
    if (valid && t < n) { node = sch[t]; b0 = brp[t]; cb = brp[t + 1] - b0; }
    const int rnode = __shfl_sync(0xffffffffu, node, ref), rcb = __shfl_sync(0xffffffffu, cb, ref);
    if (valid && (node != rnode || cb != rcb)) mism = true;
    const int mp = (rcb + 1) / 2;
    if (mp > UMP) mism = true;
    if (mp > mpw) mpw = mp;
    for (int k = 0; k < rcb && k < 2 * UMP; ++k) {
      const int nd = (valid && k < cb) ? bkv[b0 + k] : 0;
      const int rnd = __shfl_sync(0xffffffffu, nd, ref);
      if (valid && nd != rnd) mism = true;
      if (fill) {
        if (lane == 0) desc[32 * t + 4 + k] = (unsigned char)rnd;
        Lc[((long long)(kp + k / 2) * 32 + lane) * 2 + (k & 1)] = valid ? bLv[b0 + k] : 0.0;
      }
    }
    if (fill) {
      if (lane == 0) {
        for (int k = rcb; k < 28; ++k) desc[32 * t + 4 + k] = (unsigned char)P.dummy;
        *(uint32_t*)(desc + 32 * t) = (uint32_t)rnode | ((uint32_t)mp << 8) | ((uint32_t)kp << 16);
      }
      if (rcb & 1) Lc[((long long)(kp + rcb / 2) * 32 + lane) * 2 + 1] = 0.0;
      Dd[t * 32 + lane] = valid ? 1.0 / Dn[node] : 0.0;
    }
    kp += mp;
  }
  if (kp > 65535) mism = true;
  if (__any_sync(0xffffffffu, mism) && lane == 0) atomicExch(bad, 1);
  if (!fill && lane == 0) atomicMax(bad + 1, mpw);  // widest column (pairs) of any warp
  if (!fill && lane == 0) P.sizes[w] = urec_layout(S, kp).total;
  if (fill && lane == 0) *(int4*)blk = make_int4(S, kp, 0, 0);
}

// Slot order of U mode: the tile order, patches grouped by their level-0 box shape
// (each group padded to whole warps).  *ok = 0 when some warp's patches do not share
// one schedule (the caller falls back to T-records).
static int urec_build(lorpc_prec* b, int TX, int TY, cudaStream_t s, int* ok) {
  *ok = 0;
  const std::vector<int> ord = tile_order(b, TX, TY);
  const PatchGeom G = make_geom(b);
  std::map<int, std::vector<int>> groups;
  for (int j : ord) {
    if (j < 0) continue;
    int lo[3], ext[3];
    patch_box(G, j, 0, lo, ext);
    groups[ext[0] | (ext[1] << 10) | (ext[2] << 20)].push_back(j);
  }
  std::vector<int> uord;
  uord.reserve(ord.size() + 32 * groups.size());
  for (auto& g : groups) {
    uord.insert(uord.end(), g.second.begin(), g.second.end());
    uord.resize((uord.size() + 31) / 32 * 32, -1);
  }
  const long long nslots = (long long)uord.size(), nw = nslots / 32;
  if (nslots == 0) return LORPC_OK;
  LORPC_TRY(dalloc(&b->pord, uord.size()));
  LORPC_CUDA(cudaMemcpyAsync(b->pord, uord.data(), sizeof(int) * uord.size(), cudaMemcpyHostToDevice, s));
  TRecParams P{};
  P.rec = b->rec; P.recoff = b->recoff; P.pord = b->pord; P.L = b->L; P.dummy = b->max_n[0];
  long long* sizes = nullptr;
  int* bad = nullptr;
  LORPC_TRY(dalloc(&sizes, (size_t)nw));
  LORPC_TRY(dalloc(&bad, 2));
  LORPC_CUDA(cudaMemsetAsync(bad, 0, 2 * sizeof(int), s));
  P.sizes = sizes;
  const unsigned blocks = (unsigned)((nslots + 127) / 128);
  k_urec<<<blocks, 128, 0, s>>>(P, nslots, 0, bad);
  LORPC_LAUNCHED();
  std::vector<long long> h((size_t)nw);
  int hbad2[2] = {0, 0};
  LORPC_CUDA(cudaMemcpyAsync(h.data(), sizes, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaMemcpyAsync(hbad2, bad, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  const int hbad = hbad2[0];
  b->umpmax = hbad2[1];
  if (hbad) {
    dfree(sizes); dfree(bad); dfree(b->pord);
    b->pord = nullptr;
    return LORPC_OK;
  }
  long long off = 0;
  for (auto& v : h) { const long long sz = v; v = off; off += sz; }
  b->trec_bytes = off;
  LORPC_TRY(dalloc(&b->trec, (size_t)off));
  LORPC_TRY(dalloc(&b->trecoff, h.size()));
  LORPC_CUDA(cudaMemcpyAsync(b->trecoff, h.data(), sizeof(long long) * h.size(), cudaMemcpyHostToDevice, s));
  P.trec = b->trec; P.trecoff = b->trecoff;
  k_urec<<<blocks, 128, 0, s>>>(P, nslots, 1, bad);
  LORPC_LAUNCHED();
  LORPC_CUDA(cudaStreamSynchronize(s));
  dfree(sizes); dfree(bad);
  b->tslots = nslots;
  *ok = 1;
  return LORPC_OK;
}

static int tmode_finish(lorpc_prec* b, cudaStream_t s);

int trec_build(lorpc_prec* b, cudaStream_t s) {
  int TX = 32, TY = 32;  // measured on C5 (r01): 32 x 32 < 32 x 16 < 32 x 8 < lexicographic in V-cycle time
  if (const char* e = getenv("LORPC_TILE")) {  // "0": lexicographic order; "TXxTY" otherwise
    if (atoi(e) == 0) TX = TY = 1 << 30;
    else sscanf(e, "%dx%d", &TX, &TY);
  }
  // structure-only orderings (natural, RCM): one sweep schedule per warp (U-records)
  b->umode = false;
  const char* ue = getenv("LORPC_UMODE");
  if (b->desc.ordering != 0 && !b->erng && b->max_n[0] <= 254 && !(ue && atoi(ue) == 0)) {
    int ok = 0;
    LORPC_TRY(urec_build(b, TX, TY, s, &ok));
    if (ok) { b->umode = true; return tmode_finish(b, s); }
  }
  const long long nw = (b->J + 31) / 32, nslots = nw * 32;
  const std::vector<int> ord = tile_order(b, TX, TY);
  b->tslots = nslots;
  LORPC_TRY(dalloc(&b->pord, ord.size()));
  LORPC_CUDA(cudaMemcpyAsync(b->pord, ord.data(), sizeof(int) * ord.size(), cudaMemcpyHostToDevice, s));
  TRecParams P{};
  P.rec = b->rec; P.recoff = b->recoff; P.pord = b->pord; P.L = b->L; P.dummy = b->max_n[0];
  long long* sizes = nullptr;
  LORPC_TRY(dalloc(&sizes, (size_t)nw));
  P.sizes = sizes;
  const unsigned blocks = (unsigned)((nslots + 127) / 128);
  k_trec<<<blocks, 128, 0, s>>>(P, nslots, 0);
  LORPC_LAUNCHED();
  std::vector<long long> h((size_t)nw);
  LORPC_CUDA(cudaMemcpyAsync(h.data(), sizes, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  long long off = 0;
  for (auto& v : h) { const long long sz = v; v = off; off += sz; }
  b->trec_bytes = off;
  LORPC_TRY(dalloc(&b->trec, (size_t)off));
  LORPC_TRY(dalloc(&b->trecoff, h.size()));
  LORPC_CUDA(cudaMemcpyAsync(b->trecoff, h.data(), sizeof(long long) * h.size(), cudaMemcpyHostToDevice, s));
  P.trec = b->trec; P.trecoff = b->trecoff;
  k_trec<<<blocks, 128, 0, s>>>(P, nslots, 1);
  LORPC_LAUNCHED();
  LORPC_CUDA(cudaStreamSynchronize(s));
  dfree(sizes);
  return tmode_finish(b, s);
}

// packed dense coarse operators and park buffers x, y, s for the tslots warp slots of pord
static int tmode_finish(lorpc_prec* b, cudaStream_t s) {
  const long long nslots = b->tslots;
  const PatchGeom G = make_geom(b);
  const int npk = b->m->d == 3 ? TCoarse<3>::NPK : TCoarse<2>::NPK;
  LORPC_TRY(dalloc(&b->Cdi, (size_t)(nslots * npk)));
  if (b->m->d == 3) k_pack_c<3><<<nb(nslots * npk, 256), 256, 0, s>>>(b->Cd, b->Cdi, b->pord, G, nslots, b->ldc);
  else k_pack_c<2><<<nb(nslots * npk, 256), 256, 0, s>>>(b->Cd, b->Cdi, b->pord, G, nslots, b->ldc);
  LORPC_LAUNCHED();
  LORPC_CUDA(cudaStreamSynchronize(s));
  dfree(b->Cd);
  LORPC_TRY(dalloc(&b->zpark, (size_t)(nslots * 3 * b->max_n[0])));
  return LORPC_OK;
}

// ------------------------------------------------------------------ kernel
extern __shared__ __align__(16) double tsm[];

struct TcParams {
  PatchGeom G;
  const double* A0;  // finest LOR level, node-major rows of NDP doubles
  const double* W;   // separable restriction tables, level 0 -> 1
  int woff[5];
  const char* trec;
  const long long* trecoff;
  const int* pord;
  long long J, nslots;
  const double* Cp;  // [warps][NPK][32] packed dense coarse operators
  double *xpark, *ypark, *spark;  // [warp][n0max][32] x, y, s of the warp's patches (lane columns)
  int n0max;         // largest finest-level patch (= the dummy node index)
  int pfd;           // L2 prefetch distance of the sweeps (pair rows)
  int warp_doubles;
  const double* r;
  double* z;
};

__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Shared-memory layout of the warp's 32 patch vectors: node i of patch (lane) q
// at word 32 i + q: the sweeps (lanes = patches, each at its own node) are
// conflict-free for any node indices (lane q always hits bank pair q mod 16); the
// gather / scatter phases therefore also run lane = patch.  X points at the
// lane's column (word q).
#ifndef LORPC_RLD
#define LORPC_RLD __ldcs  // T-record loads (streaming)
#endif
#ifndef LORPC_PFR
#define LORPC_PFR 8  // pair rows per L2 bulk prefetch
#endif
#ifndef LORPC_XS
#define LORPC_XS 32
#endif
#define VO(i, q) ((i) * LORPC_XS + (q))

// One step's column data in registers: MP pair rows (compile-time class size)
template <int MP>
struct TStage {
  double2 l[MP > 0 ? MP : 1];
  uint32_t c[MP > 0 ? MP : 1];
};
// index pairs: IW = 1: two u8 nodes in a u16; IW = 2: two u16 nodes in a u32
template <int IW> __device__ __forceinline__ int ilo(uint32_t c) { return IW == 1 ? (c & 0xff) : (c & 0xffff); }
template <int IW> __device__ __forceinline__ int ihi(uint32_t c) { return IW == 1 ? (c >> 8) : (c >> 16); }
template <int MP, int IW>
__device__ __forceinline__ void tload(TStage<MP>& g, const double2* __restrict__ Lp, const void* __restrict__ Cp,
                                      int kp) {
#pragma unroll
  for (int p = 0; p < MP; ++p) {
    g.l[p] = LORPC_RLD(Lp + (long long)(kp + p) * 32);
    if (IW == 1) g.c[p] = LORPC_RLD((const uint16_t*)Cp + (long long)(kp + p) * 32);
    else g.c[p] = LORPC_RLD((const uint32_t*)Cp + (long long)(kp + p) * 32);
  }
}
// forward (push) step: yk = X[k]; X[i] -= L_ik yk over the column; X[k] = yk / D_k.
// All neighbour values are loaded before any is stored (the nodes of a column are
// distinct; padding entries carry L = 0 and the dummy node).
template <int MP, int IW>
__device__ __forceinline__ void tfwd_step(const TStage<MP>& g, uint32_t h, double dinv, double* X) {
  const int k = h & 0xffff;
  const double yk = X[LORPC_XS * k];
  double v0[MP > 0 ? MP : 1], v1[MP > 0 ? MP : 1];
#pragma unroll
  for (int p = 0; p < MP; ++p) { v0[p] = X[LORPC_XS * ilo<IW>(g.c[p])]; v1[p] = X[LORPC_XS * ihi<IW>(g.c[p])]; }
#pragma unroll
  for (int p = 0; p < MP; ++p) {
    X[LORPC_XS * ilo<IW>(g.c[p])] = v0[p] - g.l[p].x * yk;
    X[LORPC_XS * ihi<IW>(g.c[p])] = v1[p] - g.l[p].y * yk;
  }
  X[LORPC_XS * k] = yk * dinv;
}
// backward (pull) step: X[k] -= sum_i L_ik X[i]; four partial sums
template <int MP, int IW>
__device__ __forceinline__ void tbwd_step(const TStage<MP>& g, uint32_t h, double* X) {
  const int k = h & 0xffff;
  double a[4] = {X[LORPC_XS * k], 0.0, 0.0, 0.0};
#pragma unroll
  for (int p = 0; p < MP; ++p) {
    a[2 * (p & 1)] -= g.l[p].x * X[LORPC_XS * ilo<IW>(g.c[p])];
    a[2 * (p & 1) + 1] -= g.l[p].y * X[LORPC_XS * ihi<IW>(g.c[p])];
  }
  X[LORPC_XS * k] = (a[0] + a[1]) + (a[2] + a[3]);
}

// Sweep cursor over a T-record block (lane-adjusted pointers)
struct TSw {
  const uint32_t* H;    // header of step index 0 of the sweep order is H0; step s at H0 + s * dir
  const double* Dd;     // Dinv[t][lane] base
  const double2* Lp;    // pair rows [Kp][32] base
  const char* Cp;       // index pair rows [Kp][32] (2 * iw bytes each), lane-adjusted
  int iw;
  int S, Kp, s;         // steps, pair rows, current step (sweep order)
  int kp;               // forward: first pair row of step s; backward: one past its last
  uint32_t hc, hn;      // headers of steps s and s + 1 (0 past the end)
  int pf, TPFD, lane;   // L2 prefetch cursor / distance
};
template <bool BWD>
__device__ __forceinline__ int tstep_t(const TSw& W, int s) { return BWD ? W.S - 1 - s : s; }
template <bool BWD>
__device__ __forceinline__ void tprefetch(TSw& W, int kp) {
  if (W.lane != 0) return;
  if (!BWD) {
    while (W.pf < W.Kp && W.pf < kp + W.TPFD) {
      const int nr = min(LORPC_PFR, W.Kp - W.pf);
      l2_prefetch(W.Lp - W.lane + W.pf * 32, 512u * nr);
      l2_prefetch(W.Cp + 2 * W.iw * (W.pf * 32 - W.lane), 64u * W.iw * nr);
      W.pf += nr;
    }
  } else {
    while (W.pf > 0 && W.pf > kp - W.TPFD) {
      const int nr = min(LORPC_PFR, W.pf);
      W.pf -= nr;
      l2_prefetch(W.Lp - W.lane + W.pf * 32, 512u * nr);
      l2_prefetch(W.Cp + 2 * W.iw * (W.pf * 32 - W.lane), 64u * W.iw * nr);
    }
  }
}
__device__ __forceinline__ int mpof(uint32_t h) { return (int)(h >> 24); }

// A run of consecutive steps of class MP, one step of software pipelining (the
// next step's column is loaded while the current one is applied; the register
// stages swap roles by the two-step unroll).  Returns at a class change or the end.
template <int MP, bool BWD, int IW>
__device__ __forceinline__ void trun(TSw& W, double* X) {
  const int dir = BWD ? -32 : 32;
  if constexpr (MP > 7) {
    // wide columns (rare): no pipelining, one register stage
    for (;;) {
      TStage<MP> A;
      const int kpA = BWD ? W.kp - MP : W.kp;
      tload<MP, IW>(A, W.Lp, W.Cp, kpA);
      const double dA = BWD ? 1.0 : __ldg(W.Dd + 32 * tstep_t<BWD>(W, W.s));
      const uint32_t h2 = W.s + 2 < W.S ? __ldg(W.H + (W.s + 2) * dir) : 0u;
      tprefetch<BWD>(W, kpA);
      if (BWD) tbwd_step<MP, IW>(A, W.hc, X); else tfwd_step<MP, IW>(A, W.hc, dA, X);
      W.s += 1; W.hc = W.hn; W.hn = h2;
      W.kp = BWD ? kpA : kpA + MP;
      if (!(W.s < W.S && mpof(W.hc) == MP)) return;
    }
  }
  TStage<MP> A, B;
  int kpA = BWD ? W.kp - MP : W.kp;
  tload<MP, IW>(A, W.Lp, W.Cp, kpA);
  double dA = BWD ? 1.0 : __ldg(W.Dd + 32 * tstep_t<BWD>(W, W.s));
  for (;;) {
    // step s from A; B <- step s + 1 if it is of the same class
    const bool c1 = W.s + 1 < W.S && mpof(W.hn) == MP;
    const int kpB = BWD ? kpA - MP : kpA + MP;
    double dB = 1.0;
    if (c1) {
      tload<MP, IW>(B, W.Lp, W.Cp, kpB);
      if (!BWD) dB = __ldg(W.Dd + 32 * tstep_t<BWD>(W, W.s + 1));
    }
    uint32_t h2 = W.s + 2 < W.S ? __ldg(W.H + (W.s + 2) * dir) : 0u;
    tprefetch<BWD>(W, kpA);
    if (BWD) tbwd_step<MP, IW>(A, W.hc, X); else tfwd_step<MP, IW>(A, W.hc, dA, X);
    W.s += 1; W.hc = W.hn; W.hn = h2;
    W.kp = BWD ? kpA : kpA + MP;
    if (!c1) return;
    // step s + 1 from B; A <- step s + 2 if it is of the same class
    const bool c2 = W.s + 1 < W.S && mpof(W.hn) == MP;
    kpA = BWD ? kpB - MP : kpB + MP;
    if (c2) {
      tload<MP, IW>(A, W.Lp, W.Cp, kpA);
      if (!BWD) dA = __ldg(W.Dd + 32 * tstep_t<BWD>(W, W.s + 1));
    }
    h2 = W.s + 2 < W.S ? __ldg(W.H + (W.s + 2) * dir) : 0u;
    if (BWD) tbwd_step<MP, IW>(B, W.hc, X); else tfwd_step<MP, IW>(B, W.hc, dB, X);
    W.s += 1; W.hc = W.hn; W.hn = h2;
    W.kp = BWD ? kpB : kpB + MP;
    if (!c2) return;
  }
}

// One triangular sweep of the lane's own patch over the T-record block: forward
// (push, steps ascending, diagonal fused) or backward (pull, steps descending),
// dispatched once per run of equal step classes.  The record streams through L2
// prefetches TPFD pair rows ahead.  X = the lane's column of the warp's shared
// vectors; X[LORPC_XS * dummy] must be zero on entry to the backward sweep.
template <int NP, bool BWD, int IW>
__device__ __forceinline__ void tsweep(const char* __restrict__ blk, double* X, int TPFD, int lane) {
  const int4 hd = __ldg((const int4*)blk);
  TSw W;
  W.S = hd.x; W.Kp = hd.y;
  if (W.S == 0) return;
  const TRecLayout T = trec_layout(W.S, W.Kp, IW);
  W.iw = IW;
  W.H = (const uint32_t*)(blk + T.hdr) + lane + (BWD ? (W.S - 1) * 32 : 0);
  W.Dd = (const double*)(blk + T.D) + lane;
  W.Lp = (const double2*)(blk + T.Lc) + lane;
  W.Cp = blk + T.Ic + 2 * IW * lane;
  W.TPFD = TPFD; W.lane = lane;
  W.pf = BWD ? W.Kp : 0;
  if (lane == 0) {
    l2_prefetch((const uint32_t*)(blk + T.hdr), 128u * W.S);
    if (!BWD) l2_prefetch((const double*)(blk + T.D), 256u * W.S);
  }
  W.s = 0;
  W.kp = BWD ? W.Kp : 0;
  const int dir = BWD ? -32 : 32;
  W.hc = __ldg(W.H);
  W.hn = W.S > 1 ? __ldg(W.H + dir) : 0u;
  tprefetch<BWD>(W, W.kp);
  while (W.s < W.S) {
    switch (mpof(W.hc)) {
      case 0: trun<0, BWD, IW>(W, X); break;
      case 1: trun<1, BWD, IW>(W, X); break;
      case 2: trun<2, BWD, IW>(W, X); break;
      case 4: trun<4, BWD, IW>(W, X); break;
      case 7: if (NP >= 7) trun<(NP >= 7 ? 7 : 1), BWD, IW>(W, X); break;
      case 10: if (NP >= 10) trun<(NP >= 10 ? 10 : 1), BWD, IW>(W, X); break;
      default: if (NP >= 13) trun<(NP >= 13 ? 13 : 1), BWD, IW>(W, X); break;
    }
  }
}

// M^{-1} applied in place to the lane's column X (forward, dummy reset, backward)
template <int NP, int IW>
__device__ __forceinline__ void tsmooth(const char* __restrict__ blk, double* X, int dummy, int TPFD, int lane) {
  tsweep<NP, false, IW>(blk, X, TPFD, lane);
  X[LORPC_XS * dummy] = 0.0;
  tsweep<NP, true, IW>(blk, X, TPFD, lane);
}


// ------------------------------------------------------------------ U-mode sweeps
// The same push-forward / pull-backward sweeps as tsweep, over a U-record: step t's
// descriptor (node, pair count, column nodes) is the same in every lane (uniform
// loads, warp-uniform dispatch on the pair count, no divergence), only the values
// differ per lane.  One step of software pipelining (the next step's values and the
// descriptor two steps ahead are loaded while a step is applied); the value stream
// is prefetched into L2 TPFD pair rows ahead.
struct UDesc { uint32_t w[8]; };
__device__ __forceinline__ void uload_desc(UDesc& d, const uint4* p) {
  const uint4 a = __ldg(p), c = __ldg(p + 1);
  d.w[0] = a.x; d.w[1] = a.y; d.w[2] = a.z; d.w[3] = a.w;
  d.w[4] = c.x; d.w[5] = c.y; d.w[6] = c.z; d.w[7] = c.w;
}
__device__ __forceinline__ int unode(const UDesc& d) { return d.w[0] & 0xff; }
__device__ __forceinline__ int ump(const UDesc& d) { return (d.w[0] >> 8) & 0xff; }
__device__ __forceinline__ int ukp(const UDesc& d) { return (int)(d.w[0] >> 16); }
__device__ __forceinline__ int unb(const UDesc& d, int m) { return (d.w[1 + (m >> 2)] >> (8 * (m & 3))) & 0xff; }

template <int MPT>
struct UStage {
  double2 l[MPT];
  double dinv;
};
// the step's column: MPT predicated loads off one base address (rows of 512 bytes)
template <bool BWD, int MPT>
__device__ __forceinline__ void uload(UStage<MPT>& g, const UDesc& d, const double2* __restrict__ Lp,
                                      const double* __restrict__ Dd, int t) {
  const int mp = ump(d);
  const double2* base = Lp + (long long)ukp(d) * 32;
#pragma unroll
  for (int p = 0; p < MPT; ++p)
    if (p < mp) g.l[p] = LORPC_RLD(base + p * 32);
  if (!BWD) g.dinv = LORPC_RLD(Dd + 32 * t);
}
template <int MP, class G>
__device__ __forceinline__ void ufwd(const G& g, const UDesc& d, double* X) {
  const int k = unode(d);
  const double yk = X[LORPC_XS * k];
  double v[2 * MP + 1];
#pragma unroll
  for (int m = 0; m < 2 * MP; ++m) v[m] = X[LORPC_XS * unb(d, m)];
#pragma unroll
  for (int p = 0; p < MP; ++p) {
    X[LORPC_XS * unb(d, 2 * p)] = v[2 * p] - g.l[p].x * yk;
    X[LORPC_XS * unb(d, 2 * p + 1)] = v[2 * p + 1] - g.l[p].y * yk;
  }
  X[LORPC_XS * k] = yk * g.dinv;
}
template <int MP, class G>
__device__ __forceinline__ void ubwd(const G& g, const UDesc& d, double* X) {
  const int k = unode(d);
  double a[4] = {X[LORPC_XS * k], 0.0, 0.0, 0.0};
#pragma unroll
  for (int p = 0; p < MP; ++p) {
    a[2 * (p & 1)] -= g.l[p].x * X[LORPC_XS * unb(d, 2 * p)];
    a[2 * (p & 1) + 1] -= g.l[p].y * X[LORPC_XS * unb(d, 2 * p + 1)];
  }
  X[LORPC_XS * k] = (a[0] + a[1]) + (a[2] + a[3]);
}
template <bool BWD, int MP, class G>
__device__ __forceinline__ void ustep_mp(const G& g, const UDesc& d, double* X) {
  if (BWD) ubwd<MP>(g, d, X); else ufwd<MP>(g, d, X);
}
template <bool BWD, int MPT>
__device__ __forceinline__ void ustep(const UStage<MPT>& g, const UDesc& d, double* X) {
  constexpr int M = MPT;
  switch (ump(d)) {  // warp-uniform
    case 0: ustep_mp<BWD, 0>(g, d, X); break;
    case 1: ustep_mp<BWD, 1>(g, d, X); break;
    case 2: ustep_mp<BWD, 2>(g, d, X); break;
    case 3: ustep_mp<BWD, 3>(g, d, X); break;
    case 4: ustep_mp<BWD, 4>(g, d, X); break;
    case 5: ustep_mp<BWD, 5>(g, d, X); break;
    case 6: ustep_mp<BWD, 6>(g, d, X); break;
    case 7: ustep_mp<BWD, 7>(g, d, X); break;
    case 8: if (M >= 8) ustep_mp<BWD, (M >= 8 ? 8 : 0)>(g, d, X); break;
    case 9: if (M >= 9) ustep_mp<BWD, (M >= 9 ? 9 : 0)>(g, d, X); break;
    case 10: if (M >= 10) ustep_mp<BWD, (M >= 10 ? 10 : 0)>(g, d, X); break;
    case 11: if (M >= 11) ustep_mp<BWD, (M >= 11 ? 11 : 0)>(g, d, X); break;
    case 12: if (M >= 12) ustep_mp<BWD, (M >= 12 ? 12 : 0)>(g, d, X); break;
    default: if (M >= 13) ustep_mp<BWD, (M >= 13 ? 13 : 0)>(g, d, X); break;
  }
}
template <bool BWD, int MPT>
__device__ __forceinline__ void usweep(const char* __restrict__ blk, double* X, int TPFD, int lane) {
  const int4 hd = __ldg((const int4*)blk);
  const int S = hd.x, E2 = hd.y;
  if (S == 0) return;
  const URecLayout U = urec_layout(S, E2);
  const uint4* Dsc = (const uint4*)(blk + U.desc);
  const double* Dd = (const double*)(blk + U.D) + lane;
  const double2* Lp = (const double2*)(blk + U.Lc) + lane;
  if (lane == 0) {
    l2_prefetch(Dsc, 32u * S);
    if (!BWD) l2_prefetch(Dd - lane, 256u * S);
  }
  int pf = BWD ? E2 : 0;
  auto st = [&](int q) { return BWD ? S - 1 - q : q; };
  auto prefetch = [&](const UDesc& d) {
    if (lane != 0) return;
    if (!BWD) {
      const int kp = ukp(d);
      while (pf < E2 && pf < kp + TPFD) {
        const int nr = min(LORPC_PFR, E2 - pf);
        l2_prefetch(Lp - lane + pf * 32, 512u * nr);
        pf += nr;
      }
    } else {
      const int kp = ukp(d) + ump(d);
      while (pf > 0 && pf > kp - TPFD) {
        const int nr = min(LORPC_PFR, pf);
        pf -= nr;
        l2_prefetch(Lp - lane + pf * 32, 512u * nr);
      }
    }
  };
  UDesc dA, dB, dN;
  UStage<MPT> A, B;
  uload_desc(dA, Dsc + 2 * st(0));
  if (S > 1) uload_desc(dB, Dsc + 2 * st(1));
  uload<BWD, MPT>(A, dA, Lp, Dd, st(0));
  for (int q = 0; q < S; q += 2) {
    prefetch(dA);
    if (q + 1 < S) uload<BWD, MPT>(B, dB, Lp, Dd, st(q + 1));
    if (q + 2 < S) uload_desc(dN, Dsc + 2 * st(q + 2));
    ustep<BWD, MPT>(A, dA, X);
    if (q + 1 >= S) break;
    dA = dN;
    if (q + 2 < S) uload<BWD, MPT>(A, dA, Lp, Dd, st(q + 2));
    if (q + 3 < S) uload_desc(dN, Dsc + 2 * st(q + 3));
    ustep<BWD, MPT>(B, dB, X);
    dB = dN;
  }
}
template <int MPT>
__device__ __forceinline__ void usmooth(const char* __restrict__ blk, double* X, int dummy, int TPFD, int lane) {
  usweep<false, MPT>(blk, X, TPFD, lane);
  X[LORPC_XS * dummy] = 0.0;
  usweep<true, MPT>(blk, X, TPFD, lane);
}

// ------------------------------------------------------------------ middle phase
// Lane = patch, no shared memory; the patch vectors are the lane's columns of
// warp-interleaved global buffers [warp][node][32] (every access of a warp is one
// 256-byte row).  x: pre-smoothed iterate, y: after the coarse correction, s:
// residual handed to the post-smoothing.  The lanes of a warp walk their nodes in
// lock step; the walk runs down in z (and y) on patches of odd z (y) index, so a
// patch and its z- (y-) neighbour, one tile layer (row) apart and resident at the
// same time, read the LOR rows of their shared node planes at the same point of
// the walk, and the second read hits L2.

// 1D restriction weights of fine node (ix, iy, iz) to the coarse box (dense W[c][f],
// zero off the hat support)
template <int DIM>
__device__ __forceinline__ void tweights(const TcParams& P, const TPatch& c, int ix, int iy, int iz, double* wx,
                                         double* wy, double* wz) {
  constexpr int CX = TCoarse<DIM>::CX, CZ = TCoarse<DIM>::CZ;
  const double* Wx = P.W + P.woff[c.ec[0]];
  const double* Wy = P.W + P.woff[c.ec[1]];
  const double* Wz = P.W + P.woff[DIM == 3 ? c.ec[2] : 1];
#pragma unroll
  for (int k = 0; k < CX; ++k) {
    wx[k] = k < c.cext[0] ? __ldg(Wx + k * c.ext[0] + ix) : 0.0;
    wy[k] = k < c.cext[1] ? __ldg(Wy + k * c.ext[1] + iy) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < CZ; ++k) wz[k] = DIM == 3 ? (k < c.cext[2] ? __ldg(Wz + k * c.ext[2] + iz) : 0.0) : 1.0;
}

// one 256-bit load (LDG.E.ENL2.256): a lane-per-patch walk reads a different row in
// every lane, so each warp load costs one L1 wavefront per lane; four doubles per
// load halve the wavefronts of 16-byte loads
// LORPC_ROW_HINT: cache priority of the LOR rows (shared by neighbouring patches, against the
// streaming patch vectors and coarse operators): 0 none, 1 L2 evict-last, 2 L1 + L2 evict-last
#ifndef LORPC_ROW_HINT
#define LORPC_ROW_HINT 0
#endif
__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c, double& d) {
#if LORPC_ROW_HINT == 1
  asm volatile("ld.global.nc.L2::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
#elif LORPC_ROW_HINT == 2
  asm volatile("ld.global.nc.L1::evict_last.L2::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
#else
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
#endif
}

// s_i = r_i - (A_0 v)_i at node i of the lane's patch, v = the lane's column V
template <int DIM>
__device__ __forceinline__ double tres_node(const TcParams& P, const TPatch& c, const double* __restrict__ V, int i,
                                            int ix, int iy, int iz) {
  constexpr int ND = Dirs<DIM>::ND, NDP = Dirs<DIM>::NDP;
  const int ex = c.ext[0], ey = c.ext[1], ez = c.ext[2];
  const long long Nx = P.G.Nax[0][0], Ny = P.G.Nax[0][1];
  const unsigned gi = (unsigned)((c.lo[0] + ix) + Nx * ((c.lo[1] + iy) + Ny * (DIM == 3 ? c.lo[2] + iz : 0)));
  const uint32_t em = exist_mask<DIM>(ix, iy, iz, ex, ey, ez);
  double a0 = __ldg(P.r + gi), a1 = 0.0;
  const double* Ar = P.A0 + (size_t)gi * NDP;
  if constexpr (NDP % 4 == 0) {
#pragma unroll
    for (int d4 = 0; d4 < NDP / 4; ++d4) {
      double av[4];
      ld256(Ar + 4 * d4, av[0], av[1], av[2], av[3]);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int d = 4 * d4 + h;
        if (d >= ND) break;
        const int o = dir_dx(d) + ex * (dir_dy(d) + ey * (DIM == 3 ? dir_dz(d) : 0));
        const double v = (em & (1u << d)) ? V[(i + o) * 32] : 0.0;
        if (h & 1) a1 -= av[h] * v; else a0 -= av[h] * v;
      }
    }
  } else {
#pragma unroll
    for (int d2 = 0; d2 < NDP / 2; ++d2) {
      const double2 av = __ldg((const double2*)Ar + d2);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int d = 2 * d2 + h;
        if (d >= ND) break;
        const int o = dir_dx(d) + ex * (dir_dy(d) + ey * (DIM == 3 ? dir_dz(d) : 0));
        const double v = (em & (1u << d)) ? V[(i + o) * 32] : 0.0;
        if (h) a1 -= av.y * v; else a0 -= av.x * v;
      }
    }
  }
  return a0 + a1;
}

// node of walk step k: box coordinates with y / z reversed on odd patch rows / layers
struct TWalk {
  int ex, ey, ez, fy, fz;
  float rex, rexy;
  __device__ __forceinline__ int at(int k, int& ix, int& iy, int& iz) const {
    box_xyz(k, ex, ey, rex, rexy, ix, iy, iz);
    if (fy) iy = ey - 1 - iy;
    if (fz) iz = ez - 1 - iz;
    return ix + ex * (iy + ey * iz);
  }
};
template <int DIM>
__device__ __forceinline__ TWalk twalk(const PatchGeom& G, const TPatch& c, long long j) {
  TWalk t;
  t.ex = c.ext[0]; t.ey = c.ext[1]; t.ez = c.ext[2];
  t.rex = 1.0f / c.ext[0]; t.rexy = 1.0f / (c.ext[0] * c.ext[1]);
  const long long gx = G.kind == 0 ? G.n[0] + 1 : G.n[0], gy = G.kind == 0 ? G.n[1] + 1 : G.n[1];
  t.fy = (int)((j / gx) % gy) & 1;
  t.fz = DIM == 3 ? (int)(j / (gx * gy)) & 1 : 0;
  return t;
}

template <int DIM>
__global__ void __launch_bounds__(128) k_vt_mid(TcParams P) {
  constexpr int CX = TCoarse<DIM>::CX, CZ = TCoarse<DIM>::CZ, NC = TCoarse<DIM>::NC, NPK = TCoarse<DIM>::NPK;
  const long long slot = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (slot >= P.nslots) return;
  const long long j = P.pord[slot];
  if (j < 0) return;
  const long long w = slot >> 5;
  const int lane = threadIdx.x & 31;
  const TPatch c = tpatch<DIM>(P.G, j);
  const TWalk wk = twalk<DIM>(P.G, c, j);
  const int n0 = P.n0max;
  const long long col = w * (long long)n0 * 32 + lane;
  const double* Xp = P.xpark + col;
  double* Yp = P.ypark + col;
  double* Sp = P.spark + col;
  // s = r - A x and r_1 = P^T s (fused)
  double r1[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) r1[k] = 0.0;
  for (int k = 0; k < c.n; ++k) {
    int ix, iy, iz;
    const int f = wk.at(k, ix, iy, iz);
    const double sv = tres_node<DIM>(P, c, Xp, f, ix, iy, iz);
    double wx[CX], wy[CX], wz[CZ];
    tweights<DIM>(P, c, ix, iy, iz, wx, wy, wz);
#pragma unroll
    for (int kz = 0; kz < CZ; ++kz)
#pragma unroll
      for (int ky = 0; ky < CX; ++ky) {
        const double wv = wy[ky] * wz[kz] * sv;
#pragma unroll
        for (int kx = 0; kx < CX; ++kx) r1[kx + CX * (ky + CX * kz)] += wx[kx] * wv;
      }
  }
  // z_1 = C r_1 (packed symmetric, fixed coarse box, interleaved by lane)
  double z1[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) z1[k] = 0.0;
  {
    const double* C = P.Cp + w * 32ll * NPK + lane;
    int idx = 0;
#pragma unroll
    for (int a = 0; a < NC; ++a) {
#pragma unroll
      for (int b = a; b < NC; ++b) {
        const double cv = __ldcs(C + 32 * idx);
        z1[a] += cv * r1[b];
        if (b != a) z1[b] += cv * r1[a];
        ++idx;
      }
    }
  }
  // y = x + P z_1
  for (int k = 0; k < c.n; ++k) {
    int ix, iy, iz;
    const int f = wk.at(k, ix, iy, iz);
    double wx[CX], wy[CX], wz[CZ];
    tweights<DIM>(P, c, ix, iy, iz, wx, wy, wz);
    double t = 0.0;
#pragma unroll
    for (int kz = 0; kz < CZ; ++kz)
#pragma unroll
      for (int ky = 0; ky < CX; ++ky) {
        double u = 0.0;
#pragma unroll
        for (int kx = 0; kx < CX; ++kx) u += wx[kx] * z1[kx + CX * (ky + CX * kz)];
        t += wy[ky] * wz[kz] * u;
      }
    Yp[f * 32] = Xp[f * 32] + t;
  }
  // s = r - A y
  for (int k = 0; k < c.n; ++k) {
    int ix, iy, iz;
    const int f = wk.at(k, ix, iy, iz);
    __stcs(Sp + f * 32, tres_node<DIM>(P, c, Yp, f, ix, iy, iz));
  }
}

// 3D line variant (patch boxes of at most 5 nodes per axis, p <= 3): the lane
// walks its patch by x-lines.  For each line the 3 x 3 neighbouring lines of the
// patch vector are read once into registers (zero outside the box) and the five
// residuals use them with compile-time indices, so a node costs its LOR row (7
// 256-bit loads) and 27 FMAs instead of 27 predicated vector loads; restriction and
// prolongation are separable per line (3 FMAs per node, 27 per line).
constexpr int TLX = 5;  // largest box extent of the line variant
// park-buffer accesses of the line kernel: the patch vectors stream through once, the LOR
// rows are shared by neighbouring patches; LORPC_PARK_STREAM=1 marks the former evict-first
#ifdef LORPC_PARK_STREAM
#define LORPC_PLD(p) __ldcs(p)
#define LORPC_PST(p, v) __stcs(p, v)
#else
#define LORPC_PLD(p) (*(p))
#define LORPC_PST(p, v) (*(p) = (v))
#endif
template <bool RESTRICT>
__device__ __forceinline__ void tline_residual(const TcParams& P, const TPatch& c, const double* __restrict__ V,
                                               int iy, int iz, double* res) {
  const int ex = c.ext[0], ey = c.ext[1], ez = c.ext[2];
  const long long Nx = P.G.Nax[0][0], Ny = P.G.Nax[0][1];
  const long long g0 = c.lo[0] + Nx * ((c.lo[1] + iy) + Ny * (long long)(c.lo[2] + iz));
  // neighbouring lines (dy, dz) of V; column xx = x + 1, x in [-1, ex]
  const double* L[3][3];
  bool ok[3][3];
#pragma unroll
  for (int dz = 0; dz < 3; ++dz)
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      const int yy = iy + dy - 1, zz = iz + dz - 1;
      ok[dz][dy] = yy >= 0 && yy < ey && zz >= 0 && zz < ez;
      L[dz][dy] = V + (long long)((ok[dz][dy] ? zz * ey + yy : 0) * ex) * 32;
    }
  // columns are loaded one node ahead (column x + 2 at node x), so only a
  // 3-column window of the 3 x 3 lines is live
  double W[3][3][TLX + 2];
#pragma unroll
  for (int dz = 0; dz < 3; ++dz)
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      W[dz][dy][0] = 0.0;
      W[dz][dy][1] = ok[dz][dy] ? LORPC_PLD(L[dz][dy]) : 0.0;
    }
#pragma unroll
  for (int x = 0; x < TLX; ++x) {
    if (x >= ex) break;
#pragma unroll
    for (int dz = 0; dz < 3; ++dz)
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
        W[dz][dy][x + 2] = (ok[dz][dy] && x + 1 < ex) ? LORPC_PLD(L[dz][dy] + (x + 1) * 32) : 0.0;
    const long long gi = g0 + x;
    const double* Ar = P.A0 + (size_t)gi * 28;
    double a0 = __ldg(P.r + gi), a1 = 0.0;
#pragma unroll
    for (int d4 = 0; d4 < 7; ++d4) {
      double av[4];
      ld256(Ar + 4 * d4, av[0], av[1], av[2], av[3]);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int d = 4 * d4 + h;
        if (d >= 27) break;
        // x + 1 + dx is within [0, ex + 1]; columns past ex are zero
        const double v = (x + 2 + dir_dx(d) <= TLX + 1) ? W[dir_dz(d) + 1][dir_dy(d) + 1][x + 1 + dir_dx(d)] : 0.0;
        if (h & 1) a1 -= av[h] * v; else a0 -= av[h] * v;
      }
    }
    res[x] = a0 + a1;
  }
}

#ifndef LORPC_MID3L_MINB
#define LORPC_MID3L_MINB 1  // CTAs of 4 warps per SM asked of ptxas (1: 254 registers, 8 warps per SM)
#endif
#ifndef LORPC_MID3L_THREADS
#define LORPC_MID3L_THREADS 128  // consecutive warps (patch rows of a tile layer) per CTA
#endif
__global__ void __launch_bounds__(LORPC_MID3L_THREADS, LORPC_MID3L_MINB) k_vt_mid3l(TcParams P) {
  constexpr int NC = 27, NPK = TCoarse<3>::NPK;
  const long long slot = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (slot >= P.nslots) return;
  const long long j = P.pord[slot];
  if (j < 0) return;
  const long long w = slot >> 5;
  const int lane = threadIdx.x & 31;
  const TPatch c = tpatch<3>(P.G, j);
  const TWalk wk = twalk<3>(P.G, c, j);
  const int ex = c.ext[0], ey = c.ext[1], ez = c.ext[2];
  const long long col = w * (long long)P.n0max * 32 + lane;
  const double* Xp = P.xpark + col;
  double* Yp = P.ypark + col;
  double* Sp = P.spark + col;
  const double* Wx = P.W + P.woff[c.ec[0]];
  const double* Wy = P.W + P.woff[c.ec[1]];
  const double* Wz = P.W + P.woff[c.ec[2]];
  auto wt = [](const double* T, int k, int ce, int e, int i) { return k < ce ? __ldg(T + k * e + i) : 0.0; };
  // s = r - A x and r_1 = P^T s
  double r1[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) r1[k] = 0.0;
  for (int kz = 0; kz < ez; ++kz) {
    const int iz = wk.fz ? ez - 1 - kz : kz;
    for (int ky = 0; ky < ey; ++ky) {
      const int iy = wk.fy ? ey - 1 - ky : ky;
      double res[TLX];
      tline_residual<true>(P, c, Xp, iy, iz, res);
      double t[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int x = 0; x < TLX; ++x) {
        if (x >= ex) break;
#pragma unroll
        for (int cx = 0; cx < 3; ++cx) t[cx] += wt(Wx, cx, c.cext[0], ex, x) * res[x];
      }
      double wy[3], wz[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) { wy[k] = wt(Wy, k, c.cext[1], ey, iy); wz[k] = wt(Wz, k, c.cext[2], ez, iz); }
#pragma unroll
      for (int cz = 0; cz < 3; ++cz)
#pragma unroll
        for (int cy = 0; cy < 3; ++cy) {
          const double f = wy[cy] * wz[cz];
#pragma unroll
          for (int cx = 0; cx < 3; ++cx) r1[cx + 3 * (cy + 3 * cz)] += f * t[cx];
        }
    }
  }
  // z_1 = C r_1 (packed symmetric, fixed coarse box, interleaved by lane)
  double z1[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) z1[k] = 0.0;
  {
    const double* C = P.Cp + w * 32ll * NPK + lane;
    int idx = 0;
#pragma unroll
    for (int a = 0; a < NC; ++a) {
#pragma unroll
      for (int b = a; b < NC; ++b) {
        const double cv = __ldcs(C + 32 * idx);
        z1[a] += cv * r1[b];
        if (b != a) z1[b] += cv * r1[a];
        ++idx;
      }
    }
  }
  // y = x + P z_1, by lines
  for (int kz = 0; kz < ez; ++kz) {
    const int iz = wk.fz ? ez - 1 - kz : kz;
    for (int ky = 0; ky < ey; ++ky) {
      const int iy = wk.fy ? ey - 1 - ky : ky;
      double wy[3], wz[3], u[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < 3; ++k) { wy[k] = wt(Wy, k, c.cext[1], ey, iy); wz[k] = wt(Wz, k, c.cext[2], ez, iz); }
#pragma unroll
      for (int cz = 0; cz < 3; ++cz)
#pragma unroll
        for (int cy = 0; cy < 3; ++cy) {
          const double f = wy[cy] * wz[cz];
#pragma unroll
          for (int cx = 0; cx < 3; ++cx) u[cx] += f * z1[cx + 3 * (cy + 3 * cz)];
        }
      const long long f0 = (long long)(iz * ey + iy) * ex;
#pragma unroll
      for (int x = 0; x < TLX; ++x) {
        if (x >= ex) break;
        double e = 0.0;
#pragma unroll
        for (int cx = 0; cx < 3; ++cx) e += wt(Wx, cx, c.cext[0], ex, x) * u[cx];
        LORPC_PST(Yp + (f0 + x) * 32, LORPC_PLD(Xp + (f0 + x) * 32) + e);
      }
    }
  }
  // s = r - A y
  for (int kz = 0; kz < ez; ++kz) {
    const int iz = wk.fz ? ez - 1 - kz : kz;
    for (int ky = 0; ky < ey; ++ky) {
      const int iy = wk.fy ? ey - 1 - ky : ky;
      double res[TLX];
      tline_residual<false>(P, c, Yp, iy, iz, res);
      const long long f0 = (long long)(iz * ey + iy) * ex;
#pragma unroll
      for (int x = 0; x < TLX; ++x) {
        if (x >= ex) break;
        __stcs(Sp + (f0 + x) * 32, res[x]);
      }
    }
  }
}

// ------------------------------------------------------------------ smoothing phases
// pre (POST = false): X = r_j (gather), X = M^{-1} X, x -> xpark.
// post (POST = true): X = s (spark), X = M^{-1} X, z += I_j (y + X) (a8).
// IW = 0: U-records (one schedule per warp); IW = -1: U-records whose columns have at most 7
// pairs (smaller register stages and dispatch); IW > 0: T-records with IW-byte node indices.
template <int DIM, bool POST, int IW>
__global__ void __launch_bounds__(32) k_vt_smooth(TcParams P) {
  constexpr int NP = DIM == 3 ? 13 : 4;
  const int lane = threadIdx.x;
  const long long w = blockIdx.x;
  const int n0 = P.n0max;
  const long long jl = P.pord[w * 32 + lane];
  const bool valid = jl >= 0;
  const char* blk = P.trec + P.trecoff[w];
  const long long Nx = P.G.Nax[0][0], Ny = P.G.Nax[0][1];
  // gather / scatter lane = patch: with the unpadded layout (stride LORPC_XS = 32)
  // lanes = patches at one node are conflict-free, and the lanes' nodes of
  // x-consecutive patches are p apart in r / z
  TPatch c{};
  float rex = 1.0f, rexy = 1.0f;
  if (valid) {
    c = tpatch<DIM>(P.G, jl);
    rex = 1.0f / c.ext[0]; rexy = 1.0f / (c.ext[0] * c.ext[1]);
  }
  auto gidx = [&](int i) {
    int ix, iy, iz;
    box_xyz(i, c.ext[0], c.ext[1], rex, rexy, ix, iy, iz);
    return (c.lo[0] + ix) + Nx * ((c.lo[1] + iy) + Ny * (DIM == 3 ? c.lo[2] + iz : 0));
  };
  const long long col = w * (long long)n0 * 32 + lane;
  if (!POST) {
    // r_j = I_j^T r (a5): the box is walked x-fastest, its global index kept incrementally
    long long g = (long long)c.lo[0] + Nx * (c.lo[1] + Ny * (long long)(DIM == 3 ? c.lo[2] : 0));
    int ix = 0, iy = 0;
    for (int i = 0; i < n0; ++i) {
      const bool in = valid && i < c.n;
      tsm[VO(i, lane)] = in ? __ldg(P.r + g) : 0.0;
      ++g;
      if (++ix == c.ext[0]) {
        ix = 0; g += Nx - c.ext[0];
        if (++iy == c.ext[1]) { iy = 0; g += Nx * (Ny - c.ext[1]); }
      }
    }
  } else {
    for (int i = 0; i < n0; ++i) tsm[VO(i, lane)] = __ldcs(P.spark + col + i * 32);
  }
  tsm[VO(n0, lane)] = 0.0;  // dummy node of the padded sweep steps
  __syncwarp();
  if constexpr (IW == 0) {
    usmooth<UMP>(blk, tsm + lane, n0, P.pfd, lane);
  } else if constexpr (IW < 0) {  // U-records whose columns have at most 7 pairs
    usmooth<7>(blk, tsm + lane, n0, P.pfd, lane);
  } else {
    tsmooth<NP, IW>(blk, tsm + lane, n0, P.pfd, lane);
  }
  __syncwarp();
  if (!POST) {
    for (int i = 0; i < n0; ++i) __stcs(P.xpark + col + i * 32, tsm[VO(i, lane)]);
  } else {
    for (int i = 0; i < n0; ++i) tsm[VO(i, lane)] += __ldcs(P.ypark + col + i * 32);  // z_j = y + M^{-1} s
    if (valid)
      for (int i = 0; i < c.n; ++i) atomicAdd(P.z + gidx(i), tsm[VO(i, lane)]);  // z += I_j z_j (a8)
  }
}

static TcParams make_tparams(const lorpc_prec* b, const double* r, double* z) {
  TcParams P{};
  P.G = make_geom(b);
  P.A0 = b->lor->A[0];
  P.W = b->wtab;
  memcpy(P.woff, b->woff[0], sizeof(P.woff));
  P.trec = b->trec; P.trecoff = b->trecoff; P.pord = b->pord;
  P.J = b->J; P.nslots = b->tslots;
  P.Cp = b->Cdi;
  P.n0max = b->max_n[0];
  const long long pcol = P.nslots * b->max_n[0];
  P.xpark = b->zpark; P.ypark = b->zpark + pcol; P.spark = b->zpark + 2 * pcol;
  P.r = r; P.z = z;
  int acc = VO(b->max_n[0] + 1, 0);
  P.warp_doubles = (acc + 1) & ~1;
  P.pfd = getenv("LORPC_TPFD") ? atoi(getenv("LORPC_TPFD")) : 32;
  return P;
}

size_t tmode_smem(const lorpc_prec* b) {
  return (size_t)make_tparams(b, nullptr, nullptr).warp_doubles * sizeof(double);
}

template <int DIM, int IW>
static int tlaunch(const TcParams& P, unsigned wblocks, unsigned mblocks, size_t smem, cudaStream_t s, bool lines) {
  // the whole shared-memory carveout: C5's 32.3 KB of vectors per warp then fit 7 warps per SM
  cudaFuncSetAttribute(k_vt_smooth<DIM, false, IW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_vt_smooth<DIM, true, IW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_vt_smooth<DIM, false, IW>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_vt_smooth<DIM, true, IW>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  k_vt_smooth<DIM, false, IW><<<wblocks, 32, smem, s>>>(P);
  LORPC_LAUNCHED();
  if constexpr (DIM == 3) {
    if (lines) k_vt_mid3l<<<(unsigned)((P.nslots + LORPC_MID3L_THREADS - 1) / LORPC_MID3L_THREADS), LORPC_MID3L_THREADS, 0, s>>>(P);
    else k_vt_mid<3><<<mblocks, 128, 0, s>>>(P);
  } else {
    k_vt_mid<2><<<mblocks, 128, 0, s>>>(P);
  }
  LORPC_LAUNCHED();
  k_vt_smooth<DIM, true, IW><<<wblocks, 32, smem, s>>>(P);
  return LORPC_OK;
}

int vcycle_t_apply(const lorpc_prec* b, const double* r, double* z, cudaStream_t s) {
  const TcParams P = make_tparams(b, r, z);
  size_t smem = (size_t)P.warp_doubles * sizeof(double);
  // optional occupancy cap of the smoothing kernels (warps per SM), for L2 reuse studies
  if (const char* e = getenv("LORPC_SMOOTH_WPSM")) {
    const int wpsm = atoi(e);
    if (wpsm > 0) smem = std::max(smem, (size_t)(220 * 1024 / wpsm));
  }
  if (smem > 227 * 1024) return fail(LORPC_ERR_SIZE, "vcycle_t: warp vectors do not fit in shared memory");
  const unsigned wblocks = (unsigned)(P.nslots / 32), mblocks = (unsigned)((P.nslots + 127) / 128);
  if (b->umode) {
    const bool lines = b->m->p <= 3 && !getenv("LORPC_MID_NODEWISE");
    if (b->m->d == 2) LORPC_TRY((tlaunch<2, 0>(P, wblocks, mblocks, smem, s, false)));
    else if (b->umpmax <= 7 && !getenv("LORPC_UMP13")) LORPC_TRY((tlaunch<3, -1>(P, wblocks, mblocks, smem, s, lines)));
    else LORPC_TRY((tlaunch<3, 0>(P, wblocks, mblocks, smem, s, lines)));
  } else if (b->m->d == 2) {
    if (tiw(P.n0max) == 1) LORPC_TRY((tlaunch<2, 1>(P, wblocks, mblocks, smem, s, false)));
    else LORPC_TRY((tlaunch<2, 2>(P, wblocks, mblocks, smem, s, false)));
  } else {
    const bool lines = b->m->p <= 3 && !getenv("LORPC_MID_NODEWISE");
    if (tiw(P.n0max) == 1) LORPC_TRY((tlaunch<3, 1>(P, wblocks, mblocks, smem, s, lines)));
    else LORPC_TRY((tlaunch<3, 2>(P, wblocks, mblocks, smem, s, lines)));
  }
  LORPC_LAUNCHED();
  return LORPC_OK;
}

}  // namespace lorpc
