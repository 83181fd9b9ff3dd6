// C-ABI of libiga2l (layer L2): context setup, the Algorithm 1 schedule, CUDA-graph replay.
// Contract: include/iga2l.h.  Paper: arXiv 2009.01499 (P:<line> = /root/reference/PAPER.md).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing without a profiler attached
#include <nccl.h>   // types only; the library is dlopen'ed (the process may already hold torch's copy)

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/iga2l.h"
#include "host_setup.h"
#include "kernels.cuh"

using namespace iga2l;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CU(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? IGA2L_ENOMEM : IGA2L_ECUDA,             \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                      \
    }                                                                                       \
  } while (0)

struct DevBand {
  Band1D b{};
  int *lo = nullptr;
  double *c = nullptr;
};

struct Level {
  int64_t m = 0;
  int n = 0;          // unknowns per axis
  int64_t N = 0;      // n^d
  double *K = nullptr, *M = nullptr;   // band tables [n][2q+1]
  double *x = nullptr, *b = nullptr, *r = nullptr, *t1 = nullptr, *t2 = nullptr;
  DevBand P, PT;      // to the next coarser level: P (n x n_c), PT (n_c x n)
  DevBand Py, PTy;    // y-axis factors when the context has per-axis tables (quarter annulus)
  double *inv = nullptr;               // dense inverse at the coarsest level
  double *fdV = nullptr, *fdLam = nullptr;   // exact solve by Kronecker fast diagonalisation (large levels)
};

}  // namespace

struct iga2l_ctx {
  int dim = 2, p = 1, q = 1, s = 1, w = 0, D = 1, colours = 1;
  int ax = 0;                    // 1: per-axis 1D tables [2][n][.] (quarter annulus, A = My ⊗ Kx + Ky ⊗ Mx)
  int64_t m = 0, n1 = 0, N = 0;
  iga2l_opts opts{};
  cudaStream_t st = nullptr;
  bool own_stream = false;
  double *K1 = nullptr, *M1 = nullptr, *V = nullptr, *lam = nullptr, *g1 = nullptr;
  DevBand R, RT;
  DevBand Ry, RTy;               // y-axis transfer factors (ax = 1)
  ToeP toe{};                    // interior 1D data (A27) for the kernels' constant-bank path
  double *frags = nullptr;       // interior-block DMMA operand fragments, lane-major (A27)
  std::vector<Level> lev;
  double *r = nullptr, *t1 = nullptr, *t2 = nullptr;   // fine scratch, N each
  double *partial = nullptr, *norm = nullptr, *hist = nullptr;
  int *hist_count = nullptr;
  int npartial = 0, hist_cap = 0;
  double *hb = nullptr, *hx = nullptr, *hy = nullptr;  // staging for host pointers (fine)
  double *hcb = nullptr, *hcx = nullptr;                // staging for host pointers (coarse)
  double *pinned = nullptr;
  // graph cache: key (b, x, with_norm)
  struct G {
    const double *b = nullptr;
    double *x = nullptr;
    int norm = -1;
    cudaGraphExec_t exec = nullptr;
  } graphs[4];
  int next_graph = 0;
  int l_sm = -1;                 // first level handled by the shared-memory tail kernel
  VcLayout vcl{};
  cudaError_t launch_error = cudaSuccess;   // first failed cudaLaunchKernelEx* (reported by the next call)
  int launch_counter = 0;
  int launches_per_iter = 0;
  std::vector<void *> allocs;
  // ---- slab decomposition along the last axis; nranks > 1 ----
  // rank >= 0: one slab per process, halos / reductions over NCCL; rank == -1: all slabs live in
  // this process on this device (halo exchange = device copies) — the one-GPU test of the same path.
  int nranks = 1, rank = 0, H = 0;
  int64_t plane = 0;        // n1^{d-1}
  struct Slab {
    int z0 = 0, z1 = 0, za = 0, zb = 0;          // owned [z0, z1), stored [za, zb) (halo H each side)
    double *xp = nullptr, *bp = nullptr, *rp = nullptr, *cpart = nullptr, *t1 = nullptr, *t2 = nullptr;
    double *partial = nullptr;
    int npart = 0;
  };
  std::vector<Slab> slabs;
  void *comm = nullptr;     // ncclComm_t
  double *normparts = nullptr, *normred = nullptr;
};

namespace {

template <typename T>
int dalloc(iga2l_ctx *c, T **ptr, size_t count) {
  void *p = nullptr;
  cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) return fail(IGA2L_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  c->allocs.push_back(p);
  *ptr = static_cast<T *>(p);
  return IGA2L_OK;
}

template <typename T>
int upload(iga2l_ctx *c, T **ptr, const std::vector<T> &v) {
  int rc = dalloc(c, ptr, v.size());
  if (rc) return rc;
  CU(cudaMemcpy(*ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return IGA2L_OK;
}

int upload_band(iga2l_ctx *c, DevBand &d, const BandOp &h) {
  int rc = upload(c, &d.lo, h.lo);
  if (!rc) rc = upload(c, &d.c, h.c);
  auto span_of = [&](int t) {   // tile input span for the separable 2D transfer (t-row tiles starting
    int sp = 0;                 // at ANY row: slab views launch tiles from an arbitrary first row)
    for (int r0 = 0; r0 < h.rows; ++r0) {
      const int r1 = std::min(h.rows, r0 + t) - 1;
      sp = std::max(sp, h.lo[r1] - h.lo[r0]);
    }
    return sp;
  };
  d.b = Band1D{h.rows, h.cols, h.W, d.lo, d.c, span_of(32), span_of(16)};
  return rc;
}

int64_t ipow(int64_t a, int d) {
  int64_t r = 1;
  for (int i = 0; i < d; ++i) r *= a;
  return r;
}

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ---- launch helpers (count our kernel launches) ----
// returns the number of per-CTA partial sums the launch wrote (the count to reduce)
int L_apply(iga2l_ctx *c, const double *x, const double *b, double *y, double *partial, int mode) {
  int np = 0;
  launch_apply(c->dim, c->p, c->n1, c->K1, c->M1, x, b, y, partial, mode, c->st, &np, kFull, &c->toe,
               c->ax ? c->n1 * (2 * c->p + 1) : 0);
  c->launch_counter++;
  return np;
}

// ||b - A x||^2 -> c->norm (and hist[*count]++ if push_hist): sums exactly the partials written
void L_norm(iga2l_ctx *c, const double *x, const double *b, bool push_hist) {
  const int np = L_apply(c, x, b, c->r, c->partial, 1);
  launch_sum_partials(c->partial, np, c->norm, push_hist ? c->hist : nullptr, push_hist ? c->hist_count : nullptr,
                      c->hist_cap, c->st);
  c->launch_counter++;
}

// Tensor-product transform out = (⊗_a B) in (all axes the same 1D band B; 2D: By on the y axis if
// given), passes axis 0, 1, 2.  n_in per axis = B.cols, n_out = B.rows.  acc: add into out on the last pass.
void L_tensor(iga2l_ctx *c, int dim, const Band1D &B, const double *in, double *out, double *t1, double *t2,
              int acc, const Band1D *By = nullptr) {
  if (dim == 2) {            // one direct launch: out (+)= (By ⊗ B) in
    launch_tensor2d(in, out, B, acc, c->st, 0, -1, 0, 0, -1, 0, By);
    c->launch_counter++;
    return;
  }
  // shrinking transforms (restriction) run the last axis first, so that the contiguous-axis pass (the
  // least efficient: inner = 1) works on the smallest intermediate; growing ones (prolongation) axis 0 first
  const bool rev = B.rows < B.cols;
  const double *src = in;
  for (int k = 0; k < dim; ++k) {
    const int a = rev ? dim - 1 - k : k;
    const bool last = (k == dim - 1);
    double *dst = last ? out : (k % 2 == 0 ? t1 : t2);
    const int64_t inner = rev ? ipow(B.cols, a) : ipow(B.rows, a);
    const int64_t outer = rev ? ipow(B.rows, dim - 1 - a) : ipow(B.cols, dim - 1 - a);
    launch_band_axis(src, dst, outer, B.cols, inner, B, last ? acc : 0, c->st);
    c->launch_counter++;
    src = dst;
  }
}

void L_vcycle(iga2l_ctx *c, size_t l) {
  Level &L = c->lev[l];
  if (int(l) == c->l_sm) {                 // tail levels resident in shared memory (one cluster)
    const cudaError_t e = launch_vcycle_smem(c->dim, c->q, c->vcl, c->st);
    if (e != cudaSuccess) c->launch_error = e;
    c->launch_counter++;
    return;
  }
  if (L.fdV) {   // exact: (⊗V)(Σλ)^{-1}(⊗V)^T on the tensor pipe
    c->launch_counter += launch_coarse_fd(c->dim, L.n, L.fdV, L.fdLam, L.b, L.x, L.t1, L.t2, c->st, c->ax);
    return;
  }
  if (L.inv) {
    launch_dense_mv(int(L.N), L.inv, L.b, L.x, c->st);
    c->launch_counter++;
    return;
  }
  const int ncol = int(ipow(c->q + 1, c->dim));
  const int64_t ays = c->ax ? int64_t(L.n) * (2 * c->q + 1) : 0;   // per-axis level tables
  cudaMemsetAsync(L.x, 0, L.N * sizeof(double), c->st);   // zero initial guess (reading A13)
  for (int col = 0; col < ncol; ++col) {                 // pre-smoothing: (q+1)^d-colour GS (A11)
    launch_q_gs_colour(c->dim, c->q, L.n, L.K, L.M, L.b, L.x, col, c->st, ays);
    c->launch_counter++;
  }
  if (c->dim == 3)   // r = b - A_q x: the streaming sum-factorised operator kernel (degree q tables, no partials)
    launch_apply(3, c->q, L.n, L.K, L.M, L.x, L.b, L.r, nullptr, 1, c->st, nullptr, kFull, nullptr);
  else
    launch_q_residual(c->dim, c->q, L.n, L.K, L.M, L.b, L.x, L.r, c->st, ays);
  c->launch_counter++;
  Level &C = c->lev[l + 1];
  L_tensor(c, c->dim, L.PT.b, L.r, C.b, L.t1, L.t2, 0, c->ax ? &L.PTy.b : nullptr);   // restriction P^T (A8)
  L_vcycle(c, l + 1);
  L_tensor(c, c->dim, L.P.b, C.x, L.x, L.t1, L.t2, 1, c->ax ? &L.Py.b : nullptr);     // x += P e
  for (int col = 0; col < ncol; ++col) {                 // post-smoothing, same order
    launch_q_gs_colour(c->dim, c->q, L.n, L.K, L.M, L.b, L.x, col, c->st, ays);
    c->launch_counter++;
  }
}

// 3D: centres per z-chunk of a last-axis colour class, so that the planes one chunk's blocks touch (x) stay
// within ~mb MB of L2 across the class's D^2 colours (0: whole grid).  IGA2L_S3D_ZCHUNK_MB (read per call;
// default 0 = off): measured SLOWER at C5 (48 MB: 194 vs 179 ms per sweep; the colour kernels are not bound
// by the DRAM re-streaming, and the chunks' partial waves cost more than the L2 hits save).
int zchunk_centres(const iga2l_ctx *c) {
  const char *e = std::getenv("IGA2L_S3D_ZCHUNK_MB");
  const double mb = (e && *e) ? std::atof(e) : 0.0;
  const double plane = double(c->n1) * double(c->n1) * 8.0;
  if (c->dim != 3 || mb <= 0.0 || 2.0 * plane * double(c->n1) <= 2.0 * mb * 1048576.0) return 0;
  const int span = c->s + 2 * c->p;                              // planes of one block's window
  const int planes = int(mb * 1048576.0 / plane);
  return std::max(1, (planes - span) / c->D + 1);
}

void L_sweep(iga2l_ctx *c, const double *b, double *x, int c0, int c1) {
  const int zc = zchunk_centres(c);
  if (zc > 0) {
    // Colour-major order inside each last-axis class, chunk by chunk: blocks of one class whose centres
    // differ in z are >= D apart, hence A-decoupled across ALL the class's colours (reading A4), so this is
    // the same sweep (bitwise) with each chunk's planes L2-resident while its D^2 colours run.
    const int D = c->D, D2 = D * D;
    for (int cls = c0 / D2; cls * D2 < c1; ++cls) {
      const int a = std::max(c0, cls * D2), e = std::min(c1, (cls + 1) * D2);
      const int nz = int((c->n1 - cls + D - 1) / D);               // centres of this class
      const int nch = (nz + zc - 1) / zc, zcb = (nz + nch - 1) / nch;   // balanced chunks
      for (int k0 = 0; k0 < nz; k0 += zcb) {
        const SlabView sv{0, cls + D * k0, int(std::min<int64_t>(c->n1, cls + int64_t(D) * (k0 + zcb)))};
        for (int col = a; col < e; ++col) {
          if (!launch_schwarz_colour_fast(3, c->p, c->s, c->n1, c->K1, c->M1, c->V, c->lam, b, x, col, D, c->st, sv,
                                          c->frags, &c->toe, c->ax))
            launch_schwarz_colour(3, c->p, c->s, c->n1, c->K1, c->M1, c->V, c->lam, b, x, col, D, c->st, sv, c->ax);
          c->launch_counter++;
        }
      }
    }
    return;
  }
  for (int col = c0; col < c1; ++col) {
    if (!launch_schwarz_colour_fast(c->dim, c->p, c->s, c->n1, c->K1, c->M1, c->V, c->lam, b, x, col, c->D, c->st,
                                    kFull, c->frags, &c->toe, c->ax))
      launch_schwarz_colour(c->dim, c->p, c->s, c->n1, c->K1, c->M1, c->V, c->lam, b, x, col, c->D, c->st, kFull,
                            c->ax);
    c->launch_counter++;
  }
}

// NVTX range for the host-side scope of an API call or phase (profiler timelines; a no-op otherwise)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// One iteration of Algorithm 1, ν1 = 1, ν2 = 0.
void L_iteration(iga2l_ctx *c, const double *b, double *x, bool with_norm) {
  {
    NvtxRange r("iga2l: Schwarz sweep (D^d colours)");
    L_sweep(c, b, x, 0, c->colours);                         // u^1 = u^0 + S_p(b - A_p u^0)
  }
  const Band1D *Ry = c->ax ? &c->Ry.b : nullptr, *RTy = c->ax ? &c->RTy.b : nullptr;
  {
    NvtxRange r("iga2l: defect + restriction");
    L_apply(c, x, b, c->r, nullptr, 1);                      // d_p = b - A_p u^1
    L_tensor(c, c->dim, c->R.b, c->r, c->lev[0].b, c->t1, c->t2, 0, Ry);   // d_q = I_p^q d_p
  }
  {
    NvtxRange r("iga2l: second level");
    L_vcycle(c, 0);                                          // A_q e_q = d_q (exact or one V(1,1))
  }
  {
    NvtxRange r("iga2l: prolongation");
    L_tensor(c, c->dim, c->RT.b, c->lev[0].x, x, c->t1, c->t2, 1, RTy);   // u^1 += I_q^p e_q
  }
  if (with_norm) {
    NvtxRange r("iga2l: residual norm");
    L_norm(c, x, b, true);
  }
}

int check_ctx(const iga2l_ctx *c) {
  if (!c) return fail(IGA2L_EPARAM, "ctx is NULL");
  return IGA2L_OK;
}

// launch status after a schedule was issued: the sticky runtime error, else a recorded
// cudaLaunchKernelEx* failure (cluster launches report their configuration errors only there)
int launch_status(iga2l_ctx *c) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = c->launch_error;
  c->launch_error = cudaSuccess;
  if (e != cudaSuccess) return fail(e == cudaErrorMemoryAllocation ? IGA2L_ENOMEM : IGA2L_ECUDA,
                                    std::string("kernel launch: ") + cudaGetErrorString(e));
  return IGA2L_OK;
}

// device view of a caller vector: device pointers pass through; host pointers are staged
struct Staged {
  const double *ptr;
  bool host;
};

int stage_in(iga2l_ctx *c, const double *user, double *buf, int64_t n, Staged *out) {
  if (!user) return fail(IGA2L_EPARAM, "vector argument is NULL");
  if (is_device_ptr(user)) {
    *out = {user, false};
    return IGA2L_OK;
  }
  CU(cudaMemcpyAsync(buf, user, n * sizeof(double), cudaMemcpyHostToDevice, c->st));
  *out = {buf, true};
  return IGA2L_OK;
}

int stage_out(iga2l_ctx *c, double *user, const Staged &s, int64_t n) {
  if (s.host) {
    CU(cudaMemcpyAsync(user, s.ptr, n * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
  }
  return IGA2L_OK;
}

int run_iterations(iga2l_ctx *c, const double *b, double *x, int iters, bool with_norm) {
  if (iters <= 0) return IGA2L_OK;
  if (!c->opts.use_graph) {
    for (int k = 0; k < iters; ++k) L_iteration(c, b, x, with_norm);
    if (int rc_ = launch_status(c)) return rc_;
    return IGA2L_OK;
  }
  iga2l_ctx::G *g = nullptr;
  for (auto &gg : c->graphs)
    if (gg.exec && gg.b == b && gg.x == x && gg.norm == int(with_norm)) g = &gg;
  if (!g) {
    g = &c->graphs[c->next_graph];
    c->next_graph = (c->next_graph + 1) % 4;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    g->exec = nullptr;
    cudaGraph_t graph;
    CU(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    c->launch_counter = 0;
    L_iteration(c, b, x, with_norm);
    cudaError_t e = cudaStreamEndCapture(c->st, &graph);
    if (e != cudaSuccess) return fail(IGA2L_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    if (int rc_ = launch_status(c)) {
      cudaGraphDestroy(graph);
      return rc_;
    }
    if (!with_norm) c->launches_per_iter = c->launch_counter;
    CU(cudaGraphInstantiate(&g->exec, graph, 0));
    cudaGraphDestroy(graph);
    g->b = b;
    g->x = x;
    g->norm = int(with_norm);
  }
  for (int k = 0; k < iters; ++k) {
    NvtxRange r("iga2l: iteration (graph launch)");
    CU(cudaGraphLaunch(g->exec, c->st));
  }
  return IGA2L_OK;
}

// ------------------------------- NCCL (loaded at run time) ---------------------------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char *(*errStr)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
  static NcclApi a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return a;
#define NCCL_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name))
  NCCL_SYM(getUniqueId, "ncclGetUniqueId");
  NCCL_SYM(commInitRank, "ncclCommInitRank");
  NCCL_SYM(commDestroy, "ncclCommDestroy");
  NCCL_SYM(allReduce, "ncclAllReduce");
  NCCL_SYM(send, "ncclSend");
  NCCL_SYM(recv, "ncclRecv");
  NCCL_SYM(groupStart, "ncclGroupStart");
  NCCL_SYM(groupEnd, "ncclGroupEnd");
  NCCL_SYM(errStr, "ncclGetErrorString");
#undef NCCL_SYM
  a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.allReduce && a.send && a.recv && a.groupStart &&
         a.groupEnd && a.errStr;
  return a;
}

#define NC(call)                                                                                   \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess) return fail(IGA2L_ENCCL, std::string(#call) + ": " + nccl().errStr(r_)); \
  } while (0)

// ------------------------------- slab decomposition ----------------------------------------
// Slab bounds: balanced contiguous planes of the last axis; halo H = s - 1 + p = 2w + p planes.
void slab_bounds(int64_t n1, int R, int r, int H, int *z0, int *z1, int *za, int *zb) {
  *z0 = int(n1 * r / R);
  *z1 = int(n1 * (r + 1) / R);
  *za = std::max(0, *z0 - H);
  *zb = int(std::min<int64_t>(n1, *z1 + H));
}

// Halo exchange of a per-slab padded buffer (x or b): own boundary H planes -> neighbour halos.
int S_exchange(iga2l_ctx *c, bool which_b) {
  const int H = c->H;
  const size_t pb = size_t(c->plane) * sizeof(double);
  auto buf = [&](iga2l_ctx::Slab &s) { return which_b ? s.bp : s.xp; };
  if (c->rank < 0) {   // local mode: device copies between neighbouring slabs
    for (size_t r = 0; r + 1 < c->slabs.size(); ++r) {
      auto &A = c->slabs[r], &B = c->slabs[r + 1];
      CU(cudaMemcpyAsync(buf(B) + size_t(B.za - B.za) * c->plane, buf(A) + size_t(A.z1 - H - A.za) * c->plane,
                         H * pb, cudaMemcpyDeviceToDevice, c->st));   // A's top owned planes -> B's lower halo
      CU(cudaMemcpyAsync(buf(A) + size_t(A.z1 - A.za) * c->plane, buf(B) + size_t(B.z0 - B.za) * c->plane,
                         H * pb, cudaMemcpyDeviceToDevice, c->st));   // B's bottom owned planes -> A's upper halo
    }
    return IGA2L_OK;
  }
  auto &S = c->slabs[0];
  ncclComm_t comm = static_cast<ncclComm_t>(c->comm);
  const size_t cnt = size_t(H) * c->plane;
  NC(nccl().groupStart());
  if (c->rank > 0) {
    NC(nccl().send(buf(S) + size_t(S.z0 - S.za) * c->plane, cnt, ncclDouble, c->rank - 1, comm, c->st));
    NC(nccl().recv(buf(S), cnt, ncclDouble, c->rank - 1, comm, c->st));
  }
  if (c->rank < c->nranks - 1) {
    NC(nccl().send(buf(S) + size_t(S.z1 - H - S.za) * c->plane, cnt, ncclDouble, c->rank + 1, comm, c->st));
    NC(nccl().recv(buf(S) + size_t(S.z1 - S.za) * c->plane, cnt, ncclDouble, c->rank + 1, comm, c->st));
  }
  NC(nccl().groupEnd());
  return IGA2L_OK;
}

SlabView sv_owned(const iga2l_ctx::Slab &s) { return SlabView{s.za, s.z0, s.z1}; }

// ||b - A x||^2 over all slabs -> c->norm (and hist if given); deterministic order.
int S_norm(iga2l_ctx *c, bool push_hist) {
  for (size_t r = 0; r < c->slabs.size(); ++r) {
    auto &S = c->slabs[r];
    launch_apply(c->dim, c->p, c->n1, c->K1, c->M1, S.xp, S.bp, S.rp, S.partial, 1, c->st, &S.npart, sv_owned(S),
                 &c->toe);
    launch_sum_partials(S.partial, S.npart, c->normparts + r, nullptr, nullptr, 0, c->st);
    c->launch_counter += 2;
  }
  const double *src = c->normparts;
  int n = int(c->slabs.size());
  if (c->rank >= 0 && c->nranks > 1) {
    NC(nccl().allReduce(c->normparts, c->normred, 1, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->comm), c->st));
    src = c->normred;
    n = 1;
  }
  launch_sum_partials(src, n, c->norm, push_hist ? c->hist : nullptr, push_hist ? c->hist_count : nullptr,
                      c->hist_cap, c->st);
  c->launch_counter++;
  return IGA2L_OK;
}

// One iteration of Algorithm 1 on the slab decomposition.
int S_iteration(iga2l_ctx *c, bool with_norm) {
  const int n1 = int(c->n1), d = c->dim;
  const int per_class = int(ipow(c->D, d - 1));   // colours of one last-axis class (class outermost, A5)
  for (int zc = 0; zc < c->D; ++zc) {
    if (zc > 0)
      if (int rc = S_exchange(c, false)) return rc;   // halos current at the start of every class
    for (int k = 0; k < per_class; ++k) {
      const int col = zc * per_class + k;
      for (auto &S : c->slabs) {
        const SlabView sv{S.za, std::max(0, S.z0 - c->w), std::min(n1, S.z1 + c->w)};
        if (!launch_schwarz_colour_fast(d, c->p, c->s, c->n1, c->K1, c->M1, c->V, c->lam, S.bp, S.xp, col, c->D,
                                        c->st, sv, c->frags, &c->toe))
          launch_schwarz_colour(d, c->p, c->s, c->n1, c->K1, c->M1, c->V, c->lam, S.bp, S.xp, col, c->D, c->st, sv);
        c->launch_counter++;
      }
    }
  }
  if (int rc = S_exchange(c, false)) return rc;        // halos for the residual
  const Band1D &R = c->R.b;
  const int nc = R.rows;
  for (auto &S : c->slabs) {                           // d_p = b - A x on owned planes; partial d_q
    launch_apply(d, c->p, c->n1, c->K1, c->M1, S.xp, S.bp, S.rp, nullptr, 1, c->st, nullptr, sv_owned(S), &c->toe);
    c->launch_counter++;
    if (d == 2) {
      launch_tensor2d(S.rp, S.cpart, R, 0, c->st, S.z0, S.z1, S.za, 0, nc, 0);
      c->launch_counter++;
    } else {
      const int nz = S.z1 - S.z0;
      launch_band_axis(S.rp + size_t(S.z0 - S.za) * c->plane, S.t1, int64_t(nz) * n1, n1, 1, R, 0, c->st);
      launch_band_axis(S.t1, S.t2, nz, n1, nc, R, 0, c->st);
      launch_band_axis(S.t2, S.cpart, 1, nz, int64_t(nc) * nc, R, 0, c->st, S.z0, S.z1, S.z0);
      c->launch_counter += 3;
    }
  }
  Level &L0 = c->lev[0];
  if (c->rank < 0) {                                   // sum the slab partials in a fixed order
    CU(cudaMemcpyAsync(L0.b, c->slabs[0].cpart, L0.N * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    for (size_t r = 1; r < c->slabs.size(); ++r) {
      launch_axpy(L0.b, c->slabs[r].cpart, L0.N, c->st);
      c->launch_counter++;
    }
  } else {
    NC(nccl().allReduce(c->slabs[0].cpart, L0.b, L0.N, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->comm), c->st));
  }
  L_vcycle(c, 0);                                      // replicated second level
  for (auto &S : c->slabs) {                           // x += R^T e on owned AND halo planes
    if (d == 2) {
      launch_tensor2d(L0.x, S.xp, c->RT.b, 1, c->st, 0, nc, 0, S.za, S.zb, S.za);
      c->launch_counter++;
    } else {
      const Band1D &RT = c->RT.b;
      const int nz = S.zb - S.za;
      launch_band_axis(L0.x, S.t1, 1, nc, int64_t(nc) * nc, RT, 0, c->st, 0, -1, 0, S.za, S.zb);
      launch_band_axis(S.t1, S.t2, nz, nc, nc, RT, 0, c->st);
      launch_band_axis(S.t2, S.xp, int64_t(nz) * n1, nc, 1, RT, 1, c->st);
      c->launch_counter += 3;
    }
  }
  if (with_norm)
    if (int rc = S_norm(c, true)) return rc;
  if (int rc_ = launch_status(c)) return rc_;
  return IGA2L_OK;
}

// Caller vectors -> slab buffers.  Local mode: the caller passes the GLOBAL vectors (device);
// NCCL mode: the caller passes its owned planes [z0, z1) only; halos are then exchanged.
int S_scatter(iga2l_ctx *c, const double *b, const double *x) {
  const size_t pl = size_t(c->plane);
  for (auto &S : c->slabs) {
    if (c->rank < 0) {
      if (b) CU(cudaMemcpyAsync(S.bp, b + size_t(S.za) * pl, size_t(S.zb - S.za) * pl * 8, cudaMemcpyDeviceToDevice, c->st));
      if (x) CU(cudaMemcpyAsync(S.xp, x + size_t(S.za) * pl, size_t(S.zb - S.za) * pl * 8, cudaMemcpyDeviceToDevice, c->st));
    } else {
      if (b) CU(cudaMemcpyAsync(S.bp + size_t(S.z0 - S.za) * pl, b, size_t(S.z1 - S.z0) * pl * 8, cudaMemcpyDeviceToDevice, c->st));
      if (x) CU(cudaMemcpyAsync(S.xp + size_t(S.z0 - S.za) * pl, x, size_t(S.z1 - S.z0) * pl * 8, cudaMemcpyDeviceToDevice, c->st));
    }
  }
  if (c->rank >= 0) {
    if (b)
      if (int rc = S_exchange(c, true)) return rc;
    if (x)
      if (int rc = S_exchange(c, false)) return rc;
  }
  return IGA2L_OK;
}

int S_gather(iga2l_ctx *c, double *x) {
  const size_t pl = size_t(c->plane);
  for (auto &S : c->slabs) {
    double *dst = (c->rank < 0) ? x + size_t(S.z0) * pl : x;
    CU(cudaMemcpyAsync(dst, S.xp + size_t(S.z0 - S.za) * pl, size_t(S.z1 - S.z0) * pl * 8, cudaMemcpyDeviceToDevice,
                       c->st));
  }
  return IGA2L_OK;
}

}  // namespace

extern "C" {

const char *iga2l_last_error(void) { return g_err.c_str(); }
const char *iga2l_version(void) { return "iga2l 0.1 (sm_100a)"; }

void iga2l_default_opts(iga2l_opts *o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->coarse_mode = IGA2L_COARSE_VCYCLE;
  o->coarse_h_factor = 2;
  o->vcycle_coarsest_m = 8;
  o->stream = nullptr;
  o->use_graph = 1;
  o->nranks = 1;
  o->rank = 0;
  o->nccl_id = nullptr;
  o->geometry = IGA2L_GEOM_SQUARE;
}

int iga2l_setup(int dim, int p, int q, int64_t n, int block, int overlap, iga2l_ctx **out) {
  iga2l_opts o;
  iga2l_default_opts(&o);
  return iga2l_setup_ex(dim, p, q, n, block, overlap, &o, out);
}

int iga2l_destroy(iga2l_ctx *c) {
  if (!c) return IGA2L_OK;
  for (auto &g : c->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (c->comm) nccl().commDestroy(static_cast<ncclComm_t>(c->comm));
  for (void *p : c->allocs) cudaFree(p);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->own_stream && c->st) cudaStreamDestroy(c->st);
  delete c;
  return IGA2L_OK;
}

int iga2l_setup_ex(int dim, int p, int q, int64_t n, int block, int overlap, const iga2l_opts *opts,
                   iga2l_ctx **out) {
  if (!out) return fail(IGA2L_EPARAM, "out is NULL");
  *out = nullptr;
  iga2l_opts o;
  if (opts) o = *opts; else iga2l_default_opts(&o);
  if (dim != 2 && dim != 3) return fail(IGA2L_EPARAM, "dim must be 2 or 3");
  if (p < 1 || p > 8) return fail(IGA2L_EPARAM, "p must be in 1..8 (P:194)");
  if (q < 1 || q > 2 || q > p) return fail(IGA2L_EPARAM, "q must satisfy 1 <= q <= min(p, 2) (P:165)");
  if (n < 1 || n > 100000) return fail(IGA2L_EPARAM, "n (spans per axis) must be >= 1");
  const int64_t n1 = n + p - 2;
  if (n1 < 1) return fail(IGA2L_EPARAM, "n + p - 2 must be >= 1");
  if (block != 1 && block != 3 && block != 5 && block != 7) return fail(IGA2L_EPARAM, "block must be 1, 3, 5 or 7");
  if (block > n1) return fail(IGA2L_EPARAM, "block must be <= n + p - 2");
  if (overlap != block - 1) return fail(IGA2L_EPARAM, "overlap must be block - 1 (maximal overlap, P:186)");
  if (o.coarse_mode != IGA2L_COARSE_EXACT && o.coarse_mode != IGA2L_COARSE_VCYCLE)
    return fail(IGA2L_EPARAM, "opts.coarse_mode");
  if (o.coarse_h_factor != 1 && o.coarse_h_factor != 2) return fail(IGA2L_EPARAM, "opts.coarse_h_factor must be 1 or 2");
  if (o.coarse_h_factor == 2 && n % 2) return fail(IGA2L_EPARAM, "aggressive coarsening needs n even (S:358)");
  if (o.vcycle_coarsest_m < 1) return fail(IGA2L_EPARAM, "opts.vcycle_coarsest_m must be >= 1");
  if (o.nranks < 1) return fail(IGA2L_EPARAM, "opts.nranks must be >= 1");
  if (o.geometry != IGA2L_GEOM_SQUARE && o.geometry != IGA2L_GEOM_QUARTER_ANNULUS)
    return fail(IGA2L_EPARAM, "opts.geometry");
  const bool annulus = o.geometry == IGA2L_GEOM_QUARTER_ANNULUS;
  if (annulus && (dim != 2 || q != 2 || p < 2 || o.nranks != 1))
    return fail(IGA2L_EPARAM, "quarter annulus: dim 2, q = 2 (the geometry's degree, P:453), p >= 2, nranks 1");
  if (o.nranks == 1 && (o.rank != 0 || o.nccl_id)) return fail(IGA2L_EPARAM, "opts.rank must be 0 and opts.nccl_id NULL when nranks == 1");
  if (o.nranks > 1 && !((o.rank == -1 && !o.nccl_id) || (o.rank >= 0 && o.rank < o.nranks && o.nccl_id)))
    return fail(IGA2L_EPARAM, "opts.rank: -1 (all slabs in this process, nccl_id NULL) or 0..nranks-1 with nccl_id");
  if (o.nranks > 1) {
    const int H = block - 1 + p;
    for (int r = 0; r < o.nranks; ++r) {
      int z0, z1, za, zb;
      slab_bounds(n + p - 2, o.nranks, r, H, &z0, &z1, &za, &zb);
      if (z1 - z0 < H) return fail(IGA2L_EPARAM, "opts.nranks: every slab needs >= s - 1 + p planes (SURVEY 8(e))");
    }
  }
  const int64_t mc = n / o.coarse_h_factor;
  if (mc + q - 2 < 1) return fail(IGA2L_EPARAM, "second level is empty (n too small)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(IGA2L_ECUDA, "no CUDA device available");
  }
  const int64_t N = ipow(n1, dim);
  if (N > (int64_t)1 << 31) return fail(IGA2L_EPARAM, "problem too large");

  iga2l_ctx *c = new iga2l_ctx();
  c->dim = dim; c->p = p; c->q = q; c->s = block; c->w = (block - 1) / 2; c->D = block + p;
  c->colours = int(ipow(c->D, dim));
  c->m = n; c->n1 = n1; c->N = N; c->opts = o;
  c->ax = annulus ? 1 : 0;
  c->nranks = o.nranks;
  c->rank = o.nranks > 1 ? o.rank : 0;
  c->H = block - 1 + p;
  c->plane = ipow(n1, dim - 1);
  if (o.nranks > 1) c->opts.use_graph = 0;   // slab path: eager launches (NCCL calls in the schedule)
  auto bail = [&](int rc) { iga2l_destroy(c); return rc; };
  if (o.stream) c->st = static_cast<cudaStream_t>(o.stream);
  else {
    // blocking stream: ordered after work on the legacy default stream (safe with torch's default)
    if (cudaStreamCreate(&c->st) != cudaSuccess)
      return bail(fail(IGA2L_ECUDA, "cudaStreamCreate failed"));
    c->own_stream = true;
  }
  int rc;
  // fine level tables (P:83 via Gauss quadrature on Cox–de Boor)
  std::vector<double> K, M, V, lam;
  if (annulus) {   // per-axis weighted NURBS / B-spline tables (geometry.cpp), FD tables per axis
    annulus_band_tables(p, n, K, M);
    const size_t tw = size_t(n1) * (2 * p + 1);
    for (int a = 0; a < 2; ++a) {
      std::vector<double> Ka(K.begin() + a * tw, K.begin() + (a + 1) * tw), Ma(M.begin() + a * tw, M.begin() + (a + 1) * tw);
      std::vector<double> Va, la;
      if (!fd_tables(p, block, n1, Ka, Ma, Va, la)) return bail(fail(IGA2L_ENUMERIC, "Schwarz block matrix not SPD"));
      V.insert(V.end(), Va.begin(), Va.end());
      lam.insert(lam.end(), la.begin(), la.end());
    }
  } else {
    band_tables(p, n, K, M);
    if (!fd_tables(p, block, n1, K, M, V, lam)) return bail(fail(IGA2L_ENUMERIC, "Schwarz block matrix not SPD"));
  }
  if (!annulus) {  // interior (translation-invariant) band row and FD tables, passed to kernels by value (A27)
    int64_t tlo, thi;
    toeplitz_rows(p, n, &tlo, &thi);
    const int W = 2 * p + 1, w = (block - 1) / 2;
    if (thi - tlo >= 2 * w && W <= kToeMaxW && block <= kToeMaxS) {
      const int64_t r = (tlo + thi) / 2;
      for (int t = 0; t < W; ++t) { c->toe.k[t] = K[r * W + t]; c->toe.m[t] = M[r * W + t]; }
      for (int i = 0; i < block * block; ++i) c->toe.v[i] = V[r * block * block + i];
      for (int i = 0; i < block; ++i) c->toe.lam[i] = lam[r * block + i];
      c->toe.valid = 1;
    }
  }
  if ((rc = upload(c, &c->K1, K)) || (rc = upload(c, &c->M1, M)) || (rc = upload(c, &c->V, V)) ||
      (rc = upload(c, &c->lam, lam)) || (rc = upload(c, &c->g1, load_1d_sine(p, n))))
    return bail(rc);
  // transfers (aggressive P:263)
  for (int a = 0; a < (annulus ? 2 : 1); ++a) {
    BandOp R1 = annulus ? annulus_degree_restriction(a, p, q, n) : degree_restriction(p, q, n);
    if (o.coarse_h_factor == 2)
      R1 = multiply(transpose(annulus ? annulus_embedding(a, q, mc) : mesh_prolongation(q, mc)), R1);
    const BandOp R1T = transpose(R1);
    if (R1.W > 16 || R1T.W > 16) return bail(fail(IGA2L_EPARAM, "transfer bandwidth > 16 (p + q too large)"));
    if ((rc = upload_band(c, a ? c->Ry : c->R, R1)) || (rc = upload_band(c, a ? c->RTy : c->RT, R1T))) return bail(rc);
  }
  // second-level hierarchy
  int64_t ml = mc;
  while (true) {
    Level L;
    L.m = ml;
    L.n = int(ml + q - 2);
    L.N = ipow(L.n, dim);
    std::vector<double> Kq, Mq;
    if (annulus) annulus_band_tables(q, ml, Kq, Mq);   // [2][n][2q+1]
    else band_tables(q, ml, Kq, Mq);
    if ((rc = upload(c, &L.K, Kq)) || (rc = upload(c, &L.M, Mq)) || (rc = dalloc(c, &L.x, L.N)) ||
        (rc = dalloc(c, &L.b, L.N)) || (rc = dalloc(c, &L.r, L.N)) || (rc = dalloc(c, &L.t1, L.N)) ||
        (rc = dalloc(c, &L.t2, L.N)))
      return bail(rc);
    const bool direct = (o.coarse_mode == IGA2L_COARSE_EXACT) || ml <= o.vcycle_coarsest_m;
    const char *fde = std::getenv("IGA2L_COARSE_FD");   // force / forbid the FD exact solve (tests)
    const bool use_fd = direct && o.coarse_mode == IGA2L_COARSE_EXACT &&
                        (fde ? fde[0] == '1' : L.N > 1024) && L.n <= 2048;
    if (use_fd) {   // exact second level at any size: Kronecker fast diagonalisation (host eigensolve)
      std::vector<double> V, lam;
      if (annulus) {       // per-axis decompositions [2][n][n], [2][n]
        const size_t tw = size_t(L.n) * (2 * q + 1);
        for (int a = 0; a < 2; ++a) {
          std::vector<double> Va, la;
          if (!band_fd_tables(q, L.n, Kq.data() + a * tw, Mq.data() + a * tw, Va, la))
            return bail(fail(IGA2L_ENUMERIC, "coarse matrix not SPD"));
          V.insert(V.end(), Va.begin(), Va.end());
          lam.insert(lam.end(), la.begin(), la.end());
        }
      } else if (!coarse_fd_tables(q, ml, V, lam)) {
        return bail(fail(IGA2L_ENUMERIC, "coarse matrix not SPD"));
      }
      if ((rc = upload(c, &L.fdV, V)) || (rc = upload(c, &L.fdLam, lam))) return bail(rc);
      c->lev.push_back(L);
      break;
    }
    if (direct) {
      if (L.N > 4096) return bail(fail(IGA2L_EPARAM, "exact second level: dense inverse limited to 4096 unknowns, FD to n <= 2048 per axis"));
      std::vector<double> inv;
      if (!dense_kron_inverse(dim, q, L.n, Kq, Mq, inv, annulus ? int64_t(L.n) * (2 * q + 1) : 0))
        return bail(fail(IGA2L_ENUMERIC, "coarse matrix not SPD"));
      if ((rc = upload(c, &L.inv, inv))) return bail(rc);
      c->lev.push_back(L);
      break;
    }
    if (ml % 2) return bail(fail(IGA2L_EPARAM, "V-cycle needs the second-level m divisible by 2 down to opts.vcycle_coarsest_m"));
    BandOp P = annulus ? annulus_embedding(0, q, ml / 2) : mesh_prolongation(q, ml / 2);
    if ((rc = upload_band(c, L.P, P)) || (rc = upload_band(c, L.PT, transpose(P)))) return bail(rc);
    if (annulus) {
      BandOp Py = annulus_embedding(1, q, ml / 2);
      if ((rc = upload_band(c, L.Py, Py)) || (rc = upload_band(c, L.PTy, transpose(Py)))) return bail(rc);
    }
    c->lev.push_back(L);
    ml /= 2;
  }
  {  // level table (device pointers) for the shared-memory V-cycle tail
    std::vector<QLevelDev> tab(c->lev.size());
    for (size_t l = 0; l < c->lev.size(); ++l) {
      const Level &L = c->lev[l];
      tab[l] = QLevelDev{L.n, L.N, L.K, L.M, L.x, L.b, L.r, L.t1, L.t2, L.P.b, L.PT.b, L.inv};
    }
    // shared-memory tail (one cluster): the first (largest) level from which the rest of the cycle
    // fits, preferring the widest cluster; IGA2L_VC_SMEM=0 disables it, IGA2L_VC_FORCE_CS=<cs>
    // forces level 0 on a cluster of cs CTAs (test knob)
    const char *vc_env = std::getenv("IGA2L_VC_SMEM");
    const char *force = std::getenv("IGA2L_VC_FORCE_CS");
    // (per-axis tables: level-by-level kernels only)
    const bool want_sm = !(vc_env && vc_env[0] == '0') && c->lev.size() > 1 && !annulus;
    const size_t cap = 227 * 1024;
    for (int l0 = 0; want_sm && c->l_sm < 0 && l0 + 1 < int(c->lev.size()); ++l0) {
      VcLayout vl;
      if (force && std::atoi(force) >= 1) {
        if (vcycle_smem_layout(dim, q, tab.data(), int(tab.size()), 0, std::atoi(force), cap, &vl) &&
            vcycle_smem_probe(dim, q, vl)) { c->l_sm = 0; c->vcl = vl; }
        break;
      }
      for (int cs : {16, 8, 4, 2, 1})
        if (vcycle_smem_layout(dim, q, tab.data(), int(tab.size()), l0, cs, cap, &vl) && vcycle_smem_probe(dim, q, vl)) {
          c->l_sm = l0;
          c->vcl = vl;
          break;
        }
    }
  }
  if (dim == 2 && !annulus) {   // interior-block fragments for the DMMA colour kernel (A27)
    const int nf = export_interior_frags(p, block, n1, c->K1, c->M1, c->V, c->lam, nullptr, nullptr);
    if (nf > 0) {
      const int nc = export_centre_frags(p, block, n1, c->K1, c->M1, c->V, c->lam, nullptr, nullptr);
      if ((rc = dalloc(c, &c->frags, nf + std::max(nc, 0)))) return bail(rc);
      export_interior_frags(p, block, n1, c->K1, c->M1, c->V, c->lam, c->frags, nullptr);
      if (nc > 0) export_centre_frags(p, block, n1, c->K1, c->M1, c->V, c->lam, c->frags + nf, nullptr);
      if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(IGA2L_ECUDA, "fragment export"));
    }
  }
  c->npartial = apply_num_partials(dim, p, n1);
  if (c->nranks > 1) {   // slab buffers (padded with H halo planes) and the communicator
    const int first = c->rank < 0 ? 0 : c->rank, last = c->rank < 0 ? c->nranks - 1 : c->rank;
    for (int r = first; r <= last; ++r) {
      iga2l_ctx::Slab S;
      slab_bounds(n1, c->nranks, r, c->H, &S.z0, &S.z1, &S.za, &S.zb);
      const int64_t np = int64_t(S.zb - S.za) * c->plane;
      if ((rc = dalloc(c, &S.xp, np)) || (rc = dalloc(c, &S.bp, np)) || (rc = dalloc(c, &S.rp, np)) ||
          (rc = dalloc(c, &S.t1, np)) || (rc = dalloc(c, &S.t2, np)) || (rc = dalloc(c, &S.cpart, c->lev[0].N)) ||
          (rc = dalloc(c, &S.partial, c->npartial)))
        return bail(rc);
      c->slabs.push_back(S);
    }
    if ((rc = dalloc(c, &c->normparts, c->nranks)) || (rc = dalloc(c, &c->normred, 1))) return bail(rc);
    if (c->rank >= 0) {
      NcclApi &nc = nccl();
      if (!nc.ok) return bail(fail(IGA2L_ENCCL, "libnccl.so.2 not loadable"));
      ncclUniqueId id;
      std::memcpy(&id, o.nccl_id, sizeof(id));
      ncclComm_t comm;
      ncclResult_t r = nc.commInitRank(&comm, c->nranks, id, c->rank);
      if (r != ncclSuccess) return bail(fail(IGA2L_ENCCL, std::string("ncclCommInitRank: ") + nc.errStr(r)));
      c->comm = comm;
      c->N = int64_t(c->slabs[0].z1 - c->slabs[0].z0) * c->plane;   // caller vectors: owned planes only
    }
  }
  if ((rc = dalloc(c, &c->r, N)) || (rc = dalloc(c, &c->t1, N)) || (rc = dalloc(c, &c->t2, N)) ||
      (rc = dalloc(c, &c->partial, c->npartial)) || (rc = dalloc(c, &c->norm, 1)) ||
      (rc = dalloc(c, &c->hist_count, 1)) || (rc = dalloc(c, &c->hist, 4096)))
    return bail(rc);
  c->hist_cap = 4096;
  if (cudaMemset(c->hist_count, 0, sizeof(int)) != cudaSuccess ||
      cudaMemset(c->partial, 0, size_t(c->npartial) * sizeof(double)) != cudaSuccess)
    return bail(fail(IGA2L_ECUDA, "cudaMemset"));
  if (cudaMallocHost(&c->pinned, 64 * sizeof(double)) != cudaSuccess) return bail(fail(IGA2L_ENOMEM, "cudaMallocHost"));
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bail(fail(IGA2L_ECUDA, std::string("setup: ") + cudaGetErrorString(e)));
  if (c->nranks == 1) {  // count our kernel launches in one iteration: capture (nothing executes) and discard
    cudaGraph_t graph;
    if (cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
      return bail(fail(IGA2L_ECUDA, "capture for launch count"));
    c->launch_counter = 0;
    L_iteration(c, c->t1, c->t2, false);
    if (cudaStreamEndCapture(c->st, &graph) != cudaSuccess) return bail(fail(IGA2L_ECUDA, "end capture"));
    cudaGraphDestroy(graph);
    c->launches_per_iter = c->launch_counter;
  }
  *out = c;
  return IGA2L_OK;
}

int iga2l_sizes(const iga2l_ctx *c, int64_t *n_local, int64_t *z0, int64_t *z1, int64_t *n1) {
  if (int rc = check_ctx(c)) return rc;
  const bool one = c->nranks > 1 && c->rank >= 0;
  if (n_local) *n_local = c->N;
  if (z0) *z0 = one ? c->slabs[0].z0 : 0;
  if (z1) *z1 = one ? c->slabs[0].z1 : c->n1;
  if (n1) *n1 = c->n1;
  return IGA2L_OK;
}

int iga2l_get_info(const iga2l_ctx *c, iga2l_info *o) {
  if (int rc = check_ctx(c)) return rc;
  if (!o) return fail(IGA2L_EPARAM, "out is NULL");
  o->n1 = c->n1;
  o->N = c->N;
  o->n1c = c->lev[0].n;
  o->Nc = c->lev[0].N;
  o->colours = c->colours;
  o->levels = int(c->lev.size());
  o->launches_per_iter = c->launches_per_iter;
  // sweep = N (2k^2 + 2 SF(p,s,d)) flops, SF = sum-factorised block residual MACs,
  // or the full-stencil k (2p+1)^d where smaller.
  const double k = double(ipow(c->s, c->dim)), s = c->s, p = c->p, Wn = s + 2 * p, tp = 2 * p + 1;
  double SF = c->dim == 2 ? tp * (2 * s * Wn + 2 * s * s) : tp * (2 * s * Wn * Wn + 3 * s * s * Wn + 3 * s * s * s);
  SF = std::min(SF, k * std::pow(tp, c->dim));
  o->sweep_flops = double(c->N) * (2 * k * k + 2 * SF);
  // residual+restriction 16 B + prolongation+norm 24 B per fine DOF, ~64 B per coarse DOF
  double coarse = 0;
  for (auto &L : c->lev) coarse += double(L.N);
  o->iter_hbm_bytes = 40.0 * double(c->N) + 64.0 * coarse;
  o->vc_smem_level = c->l_sm;
  o->vc_smem_cs = c->l_sm >= 0 ? c->vcl.cs : 0;
  return IGA2L_OK;
}

int iga2l_rhs(iga2l_ctx *c, double *b) {
  if (int rc = check_ctx(c)) return rc;
  if (!c->ax) return iga2l_rhs_sine(c, b);
  if (!b) return fail(IGA2L_EPARAM, "b is NULL");
  const std::vector<double> h = annulus_load(c->p, c->m);   // host quadrature (setup-like)
  CU(cudaMemcpyAsync(b, h.data(), h.size() * sizeof(double), cudaMemcpyDefault, c->st));
  CU(cudaStreamSynchronize(c->st));
  return IGA2L_OK;
}

int iga2l_rhs_sine(iga2l_ctx *c, double *b) {
  if (int rc = check_ctx(c)) return rc;
  if (!b) return fail(IGA2L_EPARAM, "b is NULL");
  if (c->ax) return fail(IGA2L_EPARAM, "iga2l_rhs_sine: square geometry only (use iga2l_rhs)");
  const double pi = 3.14159265358979323846;
  const bool dev = is_device_ptr(b);
  if (!dev && !c->hy && dalloc(c, &c->hy, c->N)) return IGA2L_ENOMEM;
  double *dst = dev ? b : c->hy;
  if (c->nranks > 1 && c->rank >= 0) {   // owned planes of the global load vector
    double *full = nullptr;
    if (int rc = dalloc(c, &full, ipow(c->n1, c->dim))) return rc;
    launch_tensor_rhs(c->dim, c->n1, c->g1, c->dim * pi * pi, full, c->st);
    CU(cudaMemcpyAsync(dst, full + size_t(c->slabs[0].z0) * c->plane, c->N * sizeof(double), cudaMemcpyDeviceToDevice,
                       c->st));
    CU(cudaStreamSynchronize(c->st));
    c->allocs.erase(std::find(c->allocs.begin(), c->allocs.end(), (void *)full));
    cudaFree(full);
  } else {
    launch_tensor_rhs(c->dim, c->n1, c->g1, c->dim * pi * pi, dst, c->st);
  }
  if (int rc_ = launch_status(c)) return rc_;
  if (!dev) {
    CU(cudaMemcpyAsync(b, dst, c->N * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
  }
  return IGA2L_OK;
}

static int ensure_staging(iga2l_ctx *c) {
  int rc;
  if (!c->hb && (rc = dalloc(c, &c->hb, c->N))) return rc;
  if (!c->hx && (rc = dalloc(c, &c->hx, c->N))) return rc;
  if (!c->hy && (rc = dalloc(c, &c->hy, c->N))) return rc;
  if (!c->hcb && (rc = dalloc(c, &c->hcb, c->lev[0].N))) return rc;
  if (!c->hcx && (rc = dalloc(c, &c->hcx, c->lev[0].N))) return rc;
  return IGA2L_OK;
}

int iga2l_apply(iga2l_ctx *c, const double *x, double *y) {
  if (int rc = check_ctx(c)) return rc;
  if (x == y) return fail(IGA2L_EPARAM, "apply: x and y must not alias");
  if (int rc = ensure_staging(c)) return rc;
  Staged sx, sy;
  if (int rc = stage_in(c, x, c->hx, c->N, &sx)) return rc;
  if (!y) return fail(IGA2L_EPARAM, "y is NULL");
  sy = {is_device_ptr(y) ? y : c->hy, !is_device_ptr(y)};
  if (c->nranks > 1) {
    if (int rc = S_scatter(c, nullptr, sx.ptr)) return rc;
    for (auto &S : c->slabs) {
      launch_apply(c->dim, c->p, c->n1, c->K1, c->M1, S.xp, nullptr, S.rp, nullptr, 0, c->st, nullptr, sv_owned(S),
                   &c->toe);
      double *dst = const_cast<double *>(sy.ptr) + (c->rank < 0 ? size_t(S.z0) * c->plane : 0);
      CU(cudaMemcpyAsync(dst, S.rp + size_t(S.z0 - S.za) * c->plane, size_t(S.z1 - S.z0) * c->plane * 8,
                         cudaMemcpyDeviceToDevice, c->st));
    }
    if (int rc_ = launch_status(c)) return rc_;
    return stage_out(c, y, sy, c->N);
  }
  L_apply(c, sx.ptr, nullptr, const_cast<double *>(sy.ptr), nullptr, 0);
  if (int rc_ = launch_status(c)) return rc_;
  return stage_out(c, y, sy, c->N);
}

int iga2l_residual_norm(iga2l_ctx *c, const double *b, const double *x, double *out) {
  if (int rc = check_ctx(c)) return rc;
  if (!out) return fail(IGA2L_EPARAM, "out is NULL");
  if (int rc = ensure_staging(c)) return rc;
  Staged sb, sx;
  if (int rc = stage_in(c, b, c->hb, c->N, &sb)) return rc;
  if (int rc = stage_in(c, x, c->hx, c->N, &sx)) return rc;
  if (c->nranks > 1) {
    if (int rc = S_scatter(c, sb.ptr, sx.ptr)) return rc;
    if (int rc = S_norm(c, false)) return rc;
  } else {
    L_norm(c, sx.ptr, sb.ptr, false);
  }
  if (int rc_ = launch_status(c)) return rc_;
  CU(cudaMemcpyAsync(c->pinned, c->norm, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CU(cudaStreamSynchronize(c->st));
  *out = std::sqrt(c->pinned[0]);
  if (!std::isfinite(*out)) return fail(IGA2L_ENUMERIC, "residual norm is not finite");
  return IGA2L_OK;
}

int iga2l_iterate(iga2l_ctx *c, const double *b, double *x, int iters, double *res_hist) {
  NvtxRange nvtx_("iga2l_iterate");
  if (int rc = check_ctx(c)) return rc;
  if (iters < 0) return fail(IGA2L_EPARAM, "iters must be >= 0");
  if (int rc = ensure_staging(c)) return rc;
  Staged sb, sx;
  if (int rc = stage_in(c, b, c->hb, c->N, &sb)) return rc;
  if (int rc = stage_in(c, x, c->hx, c->N, &sx)) return rc;
  double *xd = const_cast<double *>(sx.ptr);
  if (res_hist && iters + 1 > c->hist_cap) return fail(IGA2L_EPARAM, "res_hist supports at most 4095 iterations per call");
  if (c->nranks > 1) {   // slab decomposition
    if (int rc = S_scatter(c, sb.ptr, xd)) return rc;
    if (res_hist) {
      CU(cudaMemsetAsync(c->hist_count, 0, sizeof(int), c->st));
      if (int rc = S_norm(c, true)) return rc;
    }
    for (int k = 0; k < iters; ++k) {
      c->launch_counter = 0;
      if (int rc = S_iteration(c, res_hist != nullptr)) return rc;
      if (!res_hist) c->launches_per_iter = c->launch_counter;
    }
    if (int rc = S_gather(c, xd)) return rc;
  } else {
    if (res_hist) {
      CU(cudaMemsetAsync(c->hist_count, 0, sizeof(int), c->st));
      L_norm(c, xd, sb.ptr, true);
    }
    if (int rc = run_iterations(c, sb.ptr, xd, iters, res_hist != nullptr)) return rc;
  }
  if (int rc_ = launch_status(c)) return rc_;
  if (res_hist) {
    CU(cudaMemcpyAsync(res_hist, c->hist, (iters + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    for (int k = 0; k <= iters; ++k)
      if (!std::isfinite(res_hist[k])) return fail(IGA2L_ENUMERIC, "residual norm is not finite");
  }
  return stage_out(c, x, sx, c->N);
}

int iga2l_lfa_torus(int dim, int p, int q, int n, int block, int h_factor, int iters, unsigned long long seed,
                    double *rho, double *ratios) {
  std::string err;
  const int rc = lfa_torus_run(dim, p, q, n, block, h_factor, iters, seed, rho, ratios, &err);
  return rc ? fail(rc, err) : IGA2L_OK;
}

int iga2l_solve(iga2l_ctx *c, const double *b, double *x, double rtol, int maxit, int *iters_out,
                double *relres_out) {
  NvtxRange nvtx_("iga2l_solve");
  if (int rc = check_ctx(c)) return rc;
  if (!(rtol > 0.0) || maxit < 0) return fail(IGA2L_EPARAM, "rtol must be > 0 and maxit >= 0");
  if (int rc = ensure_staging(c)) return rc;
  Staged sb, sx;
  if (int rc = stage_in(c, b, c->hb, c->N, &sb)) return rc;
  if (int rc = stage_in(c, x, c->hx, c->N, &sx)) return rc;
  double *xd = const_cast<double *>(sx.ptr);
  const bool slab = c->nranks > 1;
  CU(cudaMemsetAsync(c->hist_count, 0, sizeof(int), c->st));
  if (slab) {
    if (int rc = S_scatter(c, sb.ptr, xd)) return rc;
    if (int rc = S_norm(c, false)) return rc;
  } else {
    L_norm(c, xd, sb.ptr, false);
  }
  CU(cudaMemcpyAsync(c->pinned, c->norm, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CU(cudaStreamSynchronize(c->st));
  const double r0 = std::sqrt(c->pinned[0]);
  if (!std::isfinite(r0)) return fail(IGA2L_ENUMERIC, "initial residual is not finite");
  double rk = r0;
  int it = 0;
  while (it < maxit && rk > rtol * r0) {    // stop at ||r_k|| <= rtol ||r_0||
    if (slab) {
      if (int rc = S_iteration(c, true)) return rc;
    } else if (int rc = run_iterations(c, sb.ptr, xd, 1, true)) {
      return rc;
    }
    CU(cudaMemcpyAsync(c->pinned, c->norm, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    rk = std::sqrt(c->pinned[0]);
    ++it;
    if (!std::isfinite(rk)) return fail(IGA2L_ENUMERIC, "residual norm is not finite");
  }
  if (iters_out) *iters_out = it;
  if (relres_out) *relres_out = (r0 > 0) ? rk / r0 : 0.0;
  if (slab)
    if (int rc = S_gather(c, xd)) return rc;
  if (int rc = stage_out(c, x, sx, c->N)) return rc;
  if (rk > rtol * r0) return fail(IGA2L_NOTCONV, "maxit reached before rtol");
  return IGA2L_OK;
}

int iga2l_sweep(iga2l_ctx *c, const double *b, double *x, int c0, int c1) {
  NvtxRange nvtx_("iga2l_sweep");
  if (int rc = check_ctx(c)) return rc;
  if (c->nranks > 1) return fail(IGA2L_EPARAM, "phase entry points are single-domain only (nranks == 1)");
  if (c0 < 0 || c1 < c0 || c1 > c->colours) return fail(IGA2L_EPARAM, "colour range must satisfy 0 <= begin <= end <= D^d");
  if (int rc = ensure_staging(c)) return rc;
  Staged sb, sx;
  if (int rc = stage_in(c, b, c->hb, c->N, &sb)) return rc;
  if (int rc = stage_in(c, x, c->hx, c->N, &sx)) return rc;
  L_sweep(c, sb.ptr, const_cast<double *>(sx.ptr), c0, c1);
  if (int rc_ = launch_status(c)) return rc_;
  return stage_out(c, x, sx, c->N);
}

int iga2l_defect_restrict(iga2l_ctx *c, const double *b, const double *x, double *dq) {
  if (int rc = check_ctx(c)) return rc;
  if (c->nranks > 1) return fail(IGA2L_EPARAM, "phase entry points are single-domain only (nranks == 1)");
  if (int rc = ensure_staging(c)) return rc;
  Staged sb, sx;
  if (int rc = stage_in(c, b, c->hb, c->N, &sb)) return rc;
  if (int rc = stage_in(c, x, c->hx, c->N, &sx)) return rc;
  if (!dq) return fail(IGA2L_EPARAM, "dq is NULL");
  const bool dev = is_device_ptr(dq);
  double *dst = dev ? dq : c->hcb;
  L_apply(c, sx.ptr, sb.ptr, c->r, nullptr, 1);
  L_tensor(c, c->dim, c->R.b, c->r, dst, c->t1, c->t2, 0, c->ax ? &c->Ry.b : nullptr);
  if (int rc_ = launch_status(c)) return rc_;
  return stage_out(c, dq, Staged{dst, !dev}, c->lev[0].N);
}

int iga2l_coarse_solve(iga2l_ctx *c, const double *dq, double *e) {
  if (int rc = check_ctx(c)) return rc;
  if (c->nranks > 1) return fail(IGA2L_EPARAM, "phase entry points are single-domain only (nranks == 1)");
  if (int rc = ensure_staging(c)) return rc;
  if (!dq || !e) return fail(IGA2L_EPARAM, "NULL vector");
  Level &L0 = c->lev[0];
  const bool din = is_device_ptr(dq);
  CU(cudaMemcpyAsync(L0.b, dq, L0.N * sizeof(double), din ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
  L_vcycle(c, 0);
  const bool dout = is_device_ptr(e);
  CU(cudaMemcpyAsync(e, L0.x, L0.N * sizeof(double), dout ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->st));
  if (int rc_ = launch_status(c)) return rc_;
  if (!dout) CU(cudaStreamSynchronize(c->st));
  return IGA2L_OK;
}

int iga2l_prolong_add(iga2l_ctx *c, const double *e, double *x) {
  if (int rc = check_ctx(c)) return rc;
  if (c->nranks > 1) return fail(IGA2L_EPARAM, "phase entry points are single-domain only (nranks == 1)");
  if (int rc = ensure_staging(c)) return rc;
  Staged se, sx;
  if (int rc = stage_in(c, e, c->hcx, c->lev[0].N, &se)) return rc;
  if (int rc = stage_in(c, x, c->hx, c->N, &sx)) return rc;
  L_tensor(c, c->dim, c->RT.b, se.ptr, const_cast<double *>(sx.ptr), c->t1, c->t2, 1, c->ax ? &c->RTy.b : nullptr);
  if (int rc_ = launch_status(c)) return rc_;
  return stage_out(c, x, sx, c->N);
}

int iga2l_nccl_unique_id(void *out128) {
  if (!out128) return fail(IGA2L_EPARAM, "out128 is NULL");
  NcclApi &nc = nccl();
  if (!nc.ok) return fail(IGA2L_ENCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t r = nc.getUniqueId(&id);
  if (r != ncclSuccess) return fail(IGA2L_ENCCL, std::string("ncclGetUniqueId: ") + nc.errStr(r));
  std::memcpy(out128, &id, sizeof(id));
  return IGA2L_OK;
}

int iga2l_host_slab_plan(int dim, int p, int block, int64_t m, int nranks, int rank, int64_t *out8) {
  if (dim < 2 || dim > 3 || p < 1 || p > 8 || block < 1 || m < 1 || nranks < 1 || rank < 0 || rank >= nranks || !out8)
    return fail(IGA2L_EPARAM, "host_slab_plan arguments");
  const int64_t n1 = m + p - 2;
  const int H = block - 1 + p, w = (block - 1) / 2;
  int z0, z1, za, zb;
  slab_bounds(n1, nranks, rank, H, &z0, &z1, &za, &zb);
  out8[0] = z0; out8[1] = z1; out8[2] = za; out8[3] = zb;
  out8[4] = std::max<int64_t>(0, z0 - w);        // block centres handled: [out8[4], out8[5])
  out8[5] = std::min<int64_t>(n1, z1 + w);
  out8[6] = H;
  out8[7] = (z1 - z0 >= H) ? 1 : 0;              // feasible
  return IGA2L_OK;
}

int iga2l_host_coarse_fd(int q, int64_t m, double *V, double *lam) {
  if (q < 1 || q > 8 || m < 1 || m + q - 2 < 1 || m + q - 2 > 4096 || !V || !lam)
    return fail(IGA2L_EPARAM, "host_coarse_fd arguments");
  std::vector<double> v, l;
  if (!coarse_fd_tables(q, m, v, l)) return fail(IGA2L_ENUMERIC, "coarse matrix not SPD");
  std::memcpy(V, v.data(), v.size() * sizeof(double));
  std::memcpy(lam, l.data(), l.size() * sizeof(double));
  return IGA2L_OK;
}

int iga2l_host_periodic_fd(int q, int n, double *V, double *lam) {
  if (q < 1 || q > 2 || n < 2 * q + 1 || n > 4096 || !V || !lam) return fail(IGA2L_EPARAM, "host_periodic_fd arguments");
  const int64_t mb = 4 * (2 * q + 8);
  std::vector<double> Kb, Mb, v, l;
  band_tables(q, mb, Kb, Mb);
  int64_t lo, hi;
  toeplitz_rows(q, mb, &lo, &hi);
  const int64_t r = (lo + hi) / 2, W = 2 * q + 1;
  if (!periodic_fd_tables(q, n, &Kb[r * W], &Mb[r * W], v, l)) return fail(IGA2L_ENUMERIC, "periodic coarse operator");
  std::memcpy(V, v.data(), v.size() * sizeof(double));
  std::memcpy(lam, l.data(), l.size() * sizeof(double));
  return IGA2L_OK;
}

int iga2l_host_band_tables(int p, int64_t m, double *K, double *M) {
  if (p < 0 || p > 8 || m < 1 || m + p - 2 < 1 || !K || !M) return fail(IGA2L_EPARAM, "host_band_tables arguments");
  std::vector<double> k, mm;
  band_tables(p, m, k, mm);
  std::memcpy(K, k.data(), k.size() * sizeof(double));
  std::memcpy(M, mm.data(), mm.size() * sizeof(double));
  return IGA2L_OK;
}

int iga2l_host_restriction_1d(int p, int q, int64_t m, int h_factor, double *R) {
  if (p < 1 || p > 8 || q < 1 || q > p || m < 2 || (h_factor != 1 && h_factor != 2) || !R ||
      (h_factor == 2 && m % 2))
    return fail(IGA2L_EPARAM, "host_restriction_1d arguments");
  BandOp R1 = degree_restriction(p, q, m);
  if (h_factor == 2) R1 = multiply(transpose(mesh_prolongation(q, m / 2)), R1);
  for (int r = 0; r < R1.rows; ++r)
    for (int col = 0; col < R1.cols; ++col) R[(size_t)r * R1.cols + col] = R1.at(r, col);
  return IGA2L_OK;
}


int iga2l_host_annulus_tables(int p, int64_t m, double *K, double *M) {
  if (p < 2 || p > 8 || m < 1 || m + p - 2 < 1 || !K || !M) return fail(IGA2L_EPARAM, "host_annulus_tables arguments");
  std::vector<double> k, mm;
  annulus_band_tables(p, m, k, mm);
  std::memcpy(K, k.data(), k.size() * sizeof(double));
  std::memcpy(M, mm.data(), mm.size() * sizeof(double));
  return IGA2L_OK;
}

int iga2l_host_annulus_restriction_1d(int axis, int p, int q, int64_t m, int h_factor, double *R) {
  if ((axis != 0 && axis != 1) || p < 2 || p > 8 || q != 2 || q > p || m < 2 || (h_factor != 1 && h_factor != 2) ||
      !R || (h_factor == 2 && m % 2))
    return fail(IGA2L_EPARAM, "host_annulus_restriction_1d arguments");
  BandOp R1 = annulus_degree_restriction(axis, p, q, m);
  if (h_factor == 2) R1 = multiply(transpose(annulus_embedding(axis, q, m / 2)), R1);
  for (int r = 0; r < R1.rows; ++r)
    for (int col = 0; col < R1.cols; ++col) R[(size_t)r * R1.cols + col] = R1.at(r, col);
  return IGA2L_OK;
}

int iga2l_host_annulus_load(int p, int64_t m, double *b) {
  if (p < 2 || p > 8 || m < 1 || m + p - 2 < 1 || !b) return fail(IGA2L_EPARAM, "host_annulus_load arguments");
  const std::vector<double> h = annulus_load(p, m);
  std::memcpy(b, h.data(), h.size() * sizeof(double));
  return IGA2L_OK;
}

}  // extern "C"
