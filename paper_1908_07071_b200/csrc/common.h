// Internal header of the lorpc CUDA library (sm_100a, FP64).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/lorpc.h"

namespace lorpc {

constexpr int MAXP = 8;          // largest compiled polynomial degree
constexpr int MAXL = 6;          // hierarchy levels (ceil(log2 p) + 1 <= 4 for p <= 8)
constexpr int MAXC = 12;         // coarse GMG levels

// ---- error handling -------------------------------------------------------------
void set_error(const std::string& s);
int fail(int code, const std::string& s);
long long& launch_counter();
#define LORPC_CUDA(call)                                                              \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return ::lorpc::fail(LORPC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define LORPC_LAUNCHED()                                                              \
  do {                                                                                \
    ++::lorpc::launch_counter();                                                      \
    cudaError_t e_ = cudaGetLastError();                                              \
    if (e_ != cudaSuccess)                                                            \
      return ::lorpc::fail(LORPC_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
  } while (0)
#define LORPC_TRY(call)                 \
  do {                                  \
    int rc_ = (call);                   \
    if (rc_ != LORPC_OK) return rc_;    \
  } while (0)

template <class T>
int dalloc(T** p, size_t n) {
  if (n == 0) { *p = nullptr; return LORPC_OK; }
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
  if (e != cudaSuccess) return fail(LORPC_ERR_OOM, "cudaMalloc " + std::to_string(n * sizeof(T)) + " B");
  return LORPC_OK;
}
template <class T>
void dfree(T*& p) { if (p) cudaFree((void*)p); p = nullptr; }

// ---- 1D basis tables (kernel parameters; constant bank) ----------------------------
struct Basis1D {
  int p, q;
  double xi[MAXP + 1];              // GLL nodes on [0,1]
  double wq[MAXP + 1];              // volume rule weights on [0,1] (q = p+1): Gauss (reading c1) or GLL
  double xq[MAXP + 1];              // its nodes (GLL collocation: xq = xi)
  double B[(MAXP + 1) * (MAXP + 1)];  // [q][p+1]  l_j(x_q)
  double D[(MAXP + 1) * (MAXP + 1)];  // [q][p+1]  l_j'(x_q)
  double E0[MAXP + 1], E1[MAXP + 1];  // l_j'(0), l_j'(1) (face normal derivatives)
  double M1inv[(MAXP + 1) * (MAXP + 1)];  // inverse of the reference 1D mass B^T W B (BR2 lifting)
};
void make_basis(int p, Basis1D& b, int quad = 0);   // basis.cpp (quad 1: GLL collocation)
std::vector<std::vector<int>> make_chain(int p);    // basis.cpp (reading c3)

// Per-element-local 1D prolongation table between hierarchy levels l+1 -> l:
// fine local index t in [0, mf): coarse local indices c0[t], c1[t] and weights.
struct Transfer1D {
  int mf, mc, gap;
  int c0[MAXP + 1], c1[MAXP + 1];   // coarse local indices of fine local t
  double w0[MAXP + 1], w1[MAXP + 1];
  int ret[MAXP + 1];                // fine local index of coarse local index
};

struct Grid { int d; int n[3]; };  // elements per axis

}  // namespace lorpc

// ---- opaque handles -----------------------------------------------------------------
struct lorpc_mesh {
  lorpc_mesh_desc desc;
  int d, p, q, nloc, nq;            // nq = q^d
  int n[3], N[3];                   // elements / GLL nodes per axis (1 in unused axis)
  long long nel, ndof_cg, ndof, nquad, nbq;
  int ez_lo = 0, ez_hi = 0;         // CG operator: element layers [ez_lo, ez_hi) along z (3D slabs; all by default)
  lorpc::Basis1D basis;
  double* V = nullptr;              // [nvert][d]
  double* G = nullptr;              // [nel][ncomp][nq] geometric factors
  double* X = nullptr;              // [ndof_cg][d] node coordinates
  double* vol = nullptr;            // [nel] element volumes (DG)
  double* dgdiag = nullptr;         // [ndof] diag(A_IP) (DG)
  double* bq = nullptr;             // [nel][nq] coefficient b at the volume Gauss points (row f3; NULL: 1)
  double* bsub = nullptr;           // [nsub][2^d] b at the LOR subcell Gauss points (NULL: 1)
  double* ywork = nullptr;          // DG face workspace
};

struct lorpc_lor {
  const lorpc_mesh* m;
  int L;                            // hierarchy levels (finest 0)
  int ml[lorpc::MAXL];              // nodes per element per axis at level l
  int Nax[lorpc::MAXL][3];          // level node grid per axis
  long long Nl[lorpc::MAXL];
  double* A[lorpc::MAXL];           // full 3^d stencil [ND][N_l], column = node
  lorpc::Transfer1D T[lorpc::MAXL]; // T[l]: level l+1 -> l
};

struct lorpc_prec {
  const lorpc_lor* lor;
  const lorpc_mesh* m;
  lorpc_schwarz_desc desc;
  long long J;                      // patches
  int pvz0 = 0, pnvz = 0;           // vertex patches: planes [pvz0, pvz0 + pnvz) (0 = all; slab subsets)
  std::vector<short> erng_h;        // extended vertex patches: element ranges [J][6] (host; empty = default)
  short* erng = nullptr;            // the same on the device
  int emax = 2;                     // largest number of elements of a patch along an axis
  int L;
  int max_n[lorpc::MAXL];           // largest patch size per level
  char* rec = nullptr;              // per patch-level ILU records
  long long* recoff = nullptr;      // [J][L] byte offsets
  std::vector<long long> recoff_h;
  long long rec_bytes = 0;
  long long rec_max = 0;            // largest per-patch record span (bytes)
  // separable patch restriction tables: level l -> l+1, e elements along an axis
  double* wtab = nullptr;
  int woff[lorpc::MAXL][5], wfe[lorpc::MAXL][5], wce[lorpc::MAXL][5];
  int scratch_doubles = 0;          // per-patch transfer scratch (V-cycle kernel)
  int Ld = 0;                       // first level replaced by the dense coarse V-cycle operator
  double* Cd = nullptr;             // [J][ldc] dense coarse operators (column-major n_Ld x n_Ld)
  int ldc = 0;
  int lanes = 8;                    // lanes per patch in the V-cycle kernel
  // thread-per-patch V-cycle (vcycle_t.cu): warp-interleaved factors, parking buffer
  bool tmode = false;
  bool umode = false;               // thread mode with one shared sweep schedule per warp (U-records)
  int umpmax = 13;                  // widest column (pairs) of the U-records
  long long tslots = 0;             // warp slots of pord (multiple of 32)
  char* trec = nullptr;
  long long* trecoff = nullptr;
  long long trec_bytes = 0;
  double* zpark = nullptr;          // per-warp r_1 / z_1 scratch
  double* Cdi = nullptr;            // dense coarse operators, packed symmetric, interleaved by patch per warp
  int* pord = nullptr;
  // warp-per-patch fused V-cycle (vcycle_w.cu): shared-memory-staged W-records
  bool wmode = false;
  char* wrec = nullptr;
  long long* wrecoff = nullptr;     // [wslots + 1] byte offsets, slot order
  long long wrec_bytes = 0;
  int wrec_max = 0;                 // largest W-record (bytes)
  long long wslots = 0;
  double* Cq = nullptr;             // [wslots][378] packed dense coarse operators
  int wlp = 16;                     // lanes per patch of the W kernel (16: two patches per warp)
  // Q mode (vcycle_w.cu): fused V-cycle, LP lanes per patch, factors streamed through a cp.async ring
  bool qmode = false;
  int qlp = 4, qcm = 2;             // lanes per patch; ring rows (pairs per lane) per sweep step
  char* qrec = nullptr;             // per warp: {shape, S, E} | dinv[S][NPW] | values [E NPW] f64x2
  long long* qrecoff = nullptr;     // [warps] byte offsets
  long long qrec_bytes = 0;
  char* qsched = nullptr;           // per box shape: the shared sweep schedule (header + node offsets)
  int qsched_stride = 0;
  // single patch B(1) (single.cu): level-grid vectors r, z, s, w
  double* sgr[lorpc::MAXL] = {};
  double* sgz[lorpc::MAXL] = {};
  double* sgl[lorpc::MAXL] = {};
  double* sgw[lorpc::MAXL] = {};
  // coarse space (R_0)
  int nc = 0;                       // GMG levels
  int cn[lorpc::MAXC][3];           // vertices per axis
  long long cN[lorpc::MAXC];
  double* Ac[lorpc::MAXC];          // full stencil; Ac[0] aliases lor->A[L-1]
  double* dl1[lorpc::MAXC];
  double* cr[lorpc::MAXC];
  double* cz[lorpc::MAXC];
  double* cs[lorpc::MAXC];
  double* coarse_chol = nullptr;    // dense inverse of the coarsest GMG level's interior matrix
  int* coarse_idx = nullptr;        // its interior vertices (grid indices)
  int ncoarsest = 0;
  // DG workspace
  double* rcg = nullptr;
  double* zcg = nullptr;
  // PCG workspace
  double *r = nullptr, *z = nullptr, *pv = nullptr, *qv = nullptr;
  double* scal = nullptr;           // device scalars
  double* part = nullptr;           // reduction partials
  double* hostpin = nullptr;        // pinned scalars
  double* xb = nullptr;             // host-buffer solve staging (b, x)
  long long xb_n = 0;               // length the staging buffer was sized for
  cudaStream_t aux = nullptr;       // second stream (R_0 chain, concurrent with the patch batch)
  cudaEvent_t evf = nullptr, evj = nullptr;  // fork / join of the aux stream
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  long long npart = 0;              // capacity of part (reduction partials)
  // live timing of the dominant kernel (patch V-cycle), lorpc_prec_profile()
  bool prof_on = false;
  int prof_n = 0;
  std::vector<cudaEvent_t> prof_ev;
  // algorithmic byte model inputs
  long long factor_values = 0;      // sum over patch-levels of (n + nL)
};

namespace lorpc {
// internal entry points shared between translation units
int geom_setup(lorpc_mesh* m, cudaStream_t s);
int cg_apply(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s);
int cg_apply_ex(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s, bool pre, double* xy_part);
long long cg3_blocks(const lorpc_mesh* m);
int dg_apply(const lorpc_mesh* m, const double* x, double* y, cudaStream_t s);
int dg_diag_setup(lorpc_mesh* m, cudaStream_t s);
int dg_restrict_cg(const lorpc_mesh* m, const double* r_dg, double* r_cg, cudaStream_t s);
int dg_combine(const lorpc_mesh* m, const double* r_dg, const double* z_cg, double* z_dg, cudaStream_t s);
int lor_build(const lorpc_mesh* m, lorpc_lor* l, cudaStream_t s);
int schwarz_build(lorpc_prec* b, cudaStream_t s);
int gmg_build(lorpc_prec* b, double* Ac0, const int* nv, int d, cudaStream_t s);
int schwarz_apply_patches(const lorpc_prec* b, const double* r, double* z, cudaStream_t s);
int gmg_vcycle(const lorpc_prec* b, const double** out, cudaStream_t s);
int prolong_vertex_add(const lorpc_mesh* m, const double* zc, double* z, cudaStream_t s);
int schwarz_apply_cg(const lorpc_prec* b, const double* r, double* z, cudaStream_t s, double* rzpart = nullptr);
long long rz_parts(const lorpc_prec* b);  // blocks of the fused r.z partial sums (0: not fused)
int quad_points(const lorpc_mesh* m, double* xq, double* xbq, cudaStream_t s);
int subcell_points(const lorpc_mesh* m, double* xs, cudaStream_t s);
long long n_subcells(const lorpc_mesh* m);
int set_coefficient(lorpc_mesh* m, const double* bq, const double* bs, cudaStream_t s);
int rhs_assemble(const lorpc_mesh* m, const double* fq, const double* gq, double* b, cudaStream_t s);
int pcg_run(const lorpc_mesh* m, const lorpc_prec* b, const double* bvec, double* x, double rtol,
            int maxit, lorpc_pcg_report* rep, cudaStream_t s);
}  // namespace lorpc
