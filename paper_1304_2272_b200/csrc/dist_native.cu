// Native distributed Cholesky + inverse over NCCL ("the distributed variants
// gg_dist_potrf_f64 ... taking an ncclComm_t for rows, columns and the world").
//
// Replaces the factorisation loop of the reference's dist_cholesky (distgrid.py:248-288:
// element-cyclic, replicated panels all-gathered over the world) with the engine of
// distgrid.dist_potrf_inv, driven from C++: M and L 2D block-cyclic (nb) on the r x c grid of
// grid_create (distgrid.py:43-52), Cholesky FUSED with the inverse, per block column K
//   1. the owner of (K, K) factors and inverts the diagonal block (gg_potrf_f64's path); the
//      status and the nb x nb inverse are broadcast over the world communicator;
//   2. process column K % c forms the panel L_IK = A_IK L_KK^-T and broadcasts it along its
//      process ROW communicator; the panel rows a rank needs for its trailing columns are
//      assembled by one SUM all-reduce over disjoint supports along its process COLUMN;
//   3. process row K % r forms the inverse's block row X_KJ = L_KK^-1 B_KJ and broadcasts it
//      along the process column;
//   4. every rank updates its own blocks, A_IJ -= L_IK L_JK^T and B_IJ -= L_IK X_KJ (Ozaki int8
//      GEMM for the large ones, DMMA otherwise), with depth-1 look-ahead: the next block column
//      on the calling stream, the rest on a lower-priority side stream joined before the next
//      step's inverse block row.
// Collectives go either to NCCL (communicators created here from one unique id: the world, and
// the row / column communicators split from it) or to caller-provided host callbacks (the
// reference-contract transports; the tests drive several ranks on one GPU that way).
//
// NCCL is resolved at run time from the process (dlopen RTLD_NOLOAD of libnccl.so.2 -- the
// library torch already loaded -- else the system one), so the .so has no link-time NCCL
// dependency and the communicators are those of the NCCL version the process uses.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gg_internal.cuh"

namespace gg {
namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (h == nullptr) return;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    api.ok = sym(api.getUniqueId, "ncclGetUniqueId") & sym(api.commInitRank, "ncclCommInitRank") &
             sym(api.commSplit, "ncclCommSplit") & sym(api.commDestroy, "ncclCommDestroy") &
             sym(api.broadcast, "ncclBroadcast") & sym(api.allReduce, "ncclAllReduce") &
             sym(api.errorString, "ncclGetErrorString");
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const NcclApi& a = nccl();
  set_error(std::string(what) + " failed: " + (a.errorString ? a.errorString(r) : "nccl error"));
  return GG_ENCCL;
}
#define GG_NCCL_TRY(expr, what)                                  \
  do {                                                           \
    ncclResult_t _r = (expr);                                    \
    if (_r != ncclSuccess) return ::gg::nccl_fail(_r, what);     \
  } while (0)

constexpr int G_WORLD = 0, G_ROW = 1, G_COL = 2;

}  // namespace
}  // namespace gg

struct gg_dist_comms {
  int rank, nranks, r, c, pr, pc;
  bool use_nccl;
  ncclComm_t comm[3];   // world, row, column (NCCL backend)
  gg_dist_bcast_fn bcast;
  gg_dist_allreduce_fn allreduce;
  void* ctx;
};

namespace gg {
namespace {

// broadcast `bytes` bytes at dev within group g from the group member `root`
int coll_bcast(const gg_dist_comms* c, int g, void* dev, size_t bytes, int root, cudaStream_t s) {
  const int gsize = g == G_WORLD ? c->nranks : (g == G_ROW ? c->c : c->r);
  if (bytes == 0 || (gsize == 1 && !c->use_nccl)) return GG_OK;
  if (c->use_nccl) {
    GG_NCCL_TRY(nccl().broadcast(dev, dev, bytes, ncclUint8, root, c->comm[g], s), "ncclBroadcast");
    return GG_OK;
  }
  GG_CUDA_TRY(cudaStreamSynchronize(s));
  if (c->bcast(c->ctx, g, dev, bytes, root) != 0) {
    set_error("dist: broadcast callback failed");
    return GG_ENCCL;
  }
  return GG_OK;
}
// SUM all-reduce of `count` doubles at dev within group g
int coll_sum(const gg_dist_comms* c, int g, double* dev, size_t count, cudaStream_t s) {
  const int gsize = g == G_WORLD ? c->nranks : (g == G_ROW ? c->c : c->r);
  if (count == 0 || (gsize == 1 && !c->use_nccl)) return GG_OK;
  if (c->use_nccl) {
    GG_NCCL_TRY(nccl().allReduce(dev, dev, count, ncclFloat64, ncclSum, c->comm[g], s),
                "ncclAllReduce");
    return GG_OK;
  }
  GG_CUDA_TRY(cudaStreamSynchronize(s));
  if (c->allreduce(c->ctx, g, dev, count) != 0) {
    set_error("dist: all-reduce callback failed");
    return GG_ENCCL;
  }
  return GG_OK;
}

// C[m x n] = beta C + alpha A op(B) on the local shares; A column-major (lda); op(B) = B^T with
// B stored n x k (trans_b) or B stored k x n.  Large products on the Ozaki int8 GEMM.
int local_gemm(int m, int n, int k, double alpha, const double* A, long long lda, const double* B,
               long long ldb, bool trans_b, double beta, double* C, long long ldc, void* oz,
               size_t oz_bytes, cudaStream_t s) {
  if (m <= 0 || n <= 0 || k <= 0) return GG_OK;
  if (oz != nullptr && m >= 512 && n >= 512 && k >= 512 &&
      ozaki_ws_bytes(m, n, k, false) <= oz_bytes) {
    return ozaki_gemm_run(m, n, k, A, 1, lda, B, trans_b ? 1 : ldb, trans_b ? ldb : 1, C, ldc, alpha,
                          beta, 0, oz, oz_bytes, nullptr, s);
  }
  GemmArgs g{};
  g.M = m; g.N = n; g.K = k;
  g.A = A; g.lda = lda;
  g.B = B; g.ldb = ldb;
  g.C = C; g.ldc = ldc;
  g.alpha = alpha; g.beta = beta;
  return launch_dgemm(g, trans_b, s);
}

struct DistShape {
  int n, nb, nblk, r, c, pr, pc, m_loc, n_loc;
  DistShape(int n_, int nb_, const gg_dist_comms* cm) : n(n_), nb(nb_), r(cm->r), c(cm->c),
      pr(cm->pr), pc(cm->pc) {
    nblk = (n + nb - 1) / nb;
    m_loc = (pr < nblk ? (nblk - pr + r - 1) / r : 0) * nb;
    n_loc = (pc < nblk ? (nblk - pc + c - 1) / c : 0) * nb;
  }
  long long lrow(int I) const { return (long long)(I / r) * nb; }
  long long lcol(int J) const { return (long long)(J / c) * nb; }
  int rows_through(int K) const { return K < pr ? 0 : ((K - pr) / r + 1) * nb; }
  int cols_through(int K) const { return K < pc ? 0 : ((K - pc) / c + 1) * nb; }
};

inline size_t al256(size_t b) { return (b + 255) & ~size_t(255); }

struct DistWork {   // carve of the caller's workspace
  double *Dinv, *Lkk, *P[2], *Pc[2], *X;
  int* status;
  void *pws, *oz[2];
  size_t pws_bytes, oz_bytes, total;
  DistWork(const DistShape& d, char* base) {
    const size_t nb = d.nb, m = d.m_loc, nl = d.n_loc;
    size_t off = 0;
    auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += al256(bytes); return p; };
    status = reinterpret_cast<int*>(take(sizeof(int)));
    Dinv = reinterpret_cast<double*>(take(nb * nb * 8));
    Lkk = reinterpret_cast<double*>(take(nb * nb * 8));
    P[0] = reinterpret_cast<double*>(take(m * nb * 8 + 8));
    P[1] = reinterpret_cast<double*>(take(m * nb * 8 + 8));
    Pc[0] = reinterpret_cast<double*>(take(nl * nb * 8 + 8));
    Pc[1] = reinterpret_cast<double*>(take(nl * nb * 8 + 8));
    X = reinterpret_cast<double*>(take(nl * nb * 8 + 8));
    pws_bytes = potrf_ws_bytes(d.nb);
    pws = take(pws_bytes);
    const int big = m > nl ? (int)m : (int)nl;
    oz_bytes = (m >= 512 && nl >= 512) ? ozaki_ws_bytes(big, big, d.nb, false) : 0;
    oz[0] = oz_bytes ? take(oz_bytes) : nullptr;
    oz[1] = oz_bytes ? take(oz_bytes) : nullptr;
    total = off;
  }
};

__global__ void zero_block_kernel(double* A, long long lda, int rows, int cols) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)rows * cols;
       e += (long long)gridDim.x * blockDim.x)
    A[(e % rows) + (e / rows) * lda] = 0.0;
}

struct SideStream {
  cudaStream_t side = nullptr, main = nullptr;
  cudaEvent_t fork_ev = nullptr, done_ev = nullptr;
  bool pending = false;
  int open() {
    int least = 0, greatest = 0;
    GG_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    GG_CUDA_TRY(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, least));
    GG_CUDA_TRY(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    GG_CUDA_TRY(cudaEventCreateWithFlags(&done_ev, cudaEventDisableTiming));
    return GG_OK;
  }
  int fork(cudaStream_t s) {
    main = s;
    GG_CUDA_TRY(cudaEventRecord(fork_ev, s));
    GG_CUDA_TRY(cudaStreamWaitEvent(side, fork_ev, 0));
    return GG_OK;
  }
  int done() {
    GG_CUDA_TRY(cudaEventRecord(done_ev, side));
    pending = true;
    return GG_OK;
  }
  int join(cudaStream_t s) {
    if (!pending) return GG_OK;
    GG_CUDA_TRY(cudaStreamWaitEvent(s, done_ev, 0));
    pending = false;
    return GG_OK;
  }
  ~SideStream() {
    if (pending && main != nullptr) join(main);   // an early (error) return: order the caller
    if (side) cudaStreamDestroy(side);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (done_ev) cudaEventDestroy(done_ev);
  }
};

int dist_potrf_run(int n, int nb, double* A, long long lda, double* B, long long ldb,
                   const gg_dist_comms* cm, void* work, size_t work_bytes, int* info,
                   cudaStream_t s) {
  const DistShape d(n, nb, cm);
  DistWork w(d, static_cast<char*>(work));
  if (work_bytes < w.total) {
    set_error("dist_potrf: workspace too small");
    return GG_EARG;
  }
  if ((d.m_loc && lda < d.m_loc) || (d.m_loc && ldb < d.m_loc)) {
    set_error("dist_potrf: leading dimension smaller than the local row count");
    return GG_EDIM;
  }
  SideStream la;
  GG_TRY(la.open());
  for (int K = 0; K < d.nblk; ++K) {
    const int orow = K % d.r, ocol = K % d.c, owner = orow * d.c + ocol;
    int st = -1;
    if (cm->rank == owner) {
      int inf[2] = {-1, 0};
      const int rc = potrf_run(nb, A + d.lrow(K) + d.lcol(K) * lda, (int)lda, 0, w.Lkk, w.Dinv, nb,
                               w.pws, inf, s);
      if (rc == GG_ENOTPD) st = inf[0] >= 0 ? inf[0] : 0;
      else if (rc != GG_OK) return rc;
      else
        GG_CUDA_TRY(cudaMemcpy2DAsync(A + d.lrow(K) + d.lcol(K) * lda, lda * 8, w.Lkk, nb * 8,
                                      nb * 8, nb, cudaMemcpyDeviceToDevice, s));
    }
    GG_CUDA_TRY(cudaMemcpyAsync(w.status, &st, sizeof(int), cudaMemcpyHostToDevice, s));
    GG_TRY(coll_bcast(cm, G_WORLD, w.status, sizeof(int), owner, s));
    GG_CUDA_TRY(cudaMemcpyAsync(&st, w.status, sizeof(int), cudaMemcpyDeviceToHost, s));
    GG_CUDA_TRY(cudaStreamSynchronize(s));
    if (st >= 0) {
      GG_TRY(la.join(s));
      *info = K * nb + st;
      set_error("matrix not positive definite");
      return GG_ENOTPD;
    }
    GG_TRY(coll_bcast(cm, G_WORLD, w.Dinv, (size_t)nb * nb * 8, owner, s));
    const int r0 = d.rows_through(K), m_below = d.m_loc - r0;
    const int c0 = d.cols_through(K), n_right = d.n_loc - c0;
    // panels double-buffered: step K's side-stream update reads them while step K+1 forms its own
    double* P = w.P[K & 1];   // m_below x nb, ld m_below (contiguous for the broadcast)
    double* Pc = w.Pc[K & 1];
    if (m_below > 0) {
      if (d.pc == ocol) {
        GG_TRY(local_gemm(m_below, nb, nb, 1.0, A + r0 + d.lcol(K) * lda, lda, w.Dinv, nb, true,
                          0.0, P, m_below, w.oz[0], w.oz_bytes, s));
        GG_CUDA_TRY(cudaMemcpy2DAsync(A + r0 + d.lcol(K) * lda, lda * 8, P, (size_t)m_below * 8,
                                      (size_t)m_below * 8, nb, cudaMemcpyDeviceToDevice, s));
      }
      GG_TRY(coll_bcast(cm, G_ROW, P, (size_t)m_below * nb * 8, ocol, s));
    }
    if (n_right > 0) {   // panel rows of this rank's column blocks J > K (n_right x nb)
      GG_CUDA_TRY(cudaMemsetAsync(Pc, 0, (size_t)n_right * nb * 8, s));
      if (m_below > 0) {
        for (int J = K + 1; J < d.nblk; ++J) {
          if (J % d.c != d.pc || J % d.r != d.pr) continue;   // column block J also a row block
          const long long jj = d.lcol(J) - c0, ii = d.lrow(J) - r0;
          GG_CUDA_TRY(cudaMemcpy2DAsync(Pc + jj, (size_t)n_right * 8, P + ii,
                                        (size_t)m_below * 8, (size_t)nb * 8, nb,
                                        cudaMemcpyDeviceToDevice, s));
        }
      }
      GG_TRY(coll_sum(cm, G_COL, Pc, (size_t)n_right * nb, s));
    }
    GG_TRY(la.join(s));   // the previous step's side work (B's block row K, A's column K+2)
    if (c0 > 0) {   // X_KJ = Dinv B_KJ, J <= K (nb x c0, ld nb)
      if (d.pr == orow) {
        GG_TRY(local_gemm(nb, c0, nb, 1.0, w.Dinv, nb, B + d.lrow(K), ldb, false, 0.0, w.X, nb,
                          w.oz[0], w.oz_bytes, s));
        GG_CUDA_TRY(cudaMemcpy2DAsync(B + d.lrow(K), ldb * 8, w.X, (size_t)nb * 8, (size_t)nb * 8,
                                      c0, cudaMemcpyDeviceToDevice, s));
      }
      GG_TRY(coll_bcast(cm, G_COL, w.X, (size_t)nb * c0 * 8, orow, s));
    }
    if (m_below == 0) continue;
    const int nxt = (n_right > 0 && (K + 1) % d.c == d.pc) ? nb : 0;
    if (nxt)
      GG_TRY(local_gemm(m_below, nxt, nb, -1.0, P, m_below, Pc, n_right, true, 1.0,
                        A + r0 + c0 * lda, lda, w.oz[0], w.oz_bytes, s));
    GG_TRY(la.fork(s));
    if (n_right > nxt)
      GG_TRY(local_gemm(m_below, n_right - nxt, nb, -1.0, P, m_below, Pc + nxt, n_right, true,
                        1.0, A + r0 + (c0 + nxt) * lda, lda, w.oz[1], w.oz_bytes, la.side));
    if (c0 > 0)
      GG_TRY(local_gemm(m_below, c0, nb, -1.0, P, m_below, w.X, nb, false, 1.0, B + r0, ldb,
                        w.oz[1], w.oz_bytes, la.side));
    GG_TRY(la.done());
  }
  GG_TRY(la.join(s));
  // strictly upper blocks of the factor's share: zero (L is lower triangular)
  for (int J = d.pc; J < d.nblk; J += d.c)
    for (int I = d.pr; I < J; I += d.r) {
      zero_block_kernel<<<64, 256, 0, s>>>(A + d.lrow(I) + d.lcol(J) * lda, lda, nb, nb);
      GG_LAUNCH_CHECK("zero_block_kernel");
    }
  return GG_OK;
}

__global__ void sub_block_kernel(int rows, int cols, const double* __restrict__ X, long long ldx,
                                 const double* __restrict__ P, long long ldp,
                                 double* __restrict__ R) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e % rows, j = e / rows;
    R[e] = X[i + j * ldx] - P[i + j * ldp];
  }
}

struct TrsmWork {   // carve of the caller's workspace for dist_trsm_run
  double *Xg, *part, *rhs, *xk, *Lkk, *Dinv;
  void* tws;
  size_t tws_bytes, total;
  TrsmWork(const DistShape& d, int k, char* base) {
    const size_t nb = d.nb, kk = k > 0 ? k : 1;
    size_t off = 0;
    auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += al256(bytes); return p; };
    Xg = reinterpret_cast<double*>(take((size_t)d.n_loc * kk * 8 + 8));
    part = reinterpret_cast<double*>(take(nb * kk * 8));
    rhs = reinterpret_cast<double*>(take(nb * kk * 8));
    xk = reinterpret_cast<double*>(take(nb * kk * 8));
    Lkk = reinterpret_cast<double*>(take(nb * nb * 8));
    Dinv = reinterpret_cast<double*>(take(nb * nb * 8));
    tws_bytes = trtri_ws_bytes(d.nb);
    tws = take(tws_bytes);
    total = off;
  }
};

// X = L^-1 X for a block-cyclic lower-triangular L and a replicated right-hand side X (n_pad x k,
// ld ldx): blocked forward substitution over the block rows K,
//   X_K = L_KK^-1 (X_K - sum_{J<K} L_KJ X_J),
// process row K%r forms the partial product of its column blocks J < K (the rows X_J it needs are
// kept gathered in Xg as they are solved), one SUM all-reduce along the process row, the owner of
// (K, K) applies its diagonal block's inverse and broadcasts X_K over the world.
int dist_trsm_run(int n, int nb, int k, const double* L, long long lda, double* X, long long ldx,
                  const gg_dist_comms* cm, void* work, size_t work_bytes, cudaStream_t s) {
  const DistShape d(n, nb, cm);
  TrsmWork w(d, k, static_cast<char*>(work));
  if (work_bytes < w.total) {
    set_error("dist_trsm: workspace too small");
    return GG_EARG;
  }
  if (ldx < (long long)d.nblk * nb || (d.m_loc && lda < d.m_loc)) {
    set_error("dist_trsm: leading dimension too small (ldx >= padded n, lda >= m_loc)");
    return GG_EDIM;
  }
  if (k <= 0) return GG_OK;
  int ng = 0;   // local column blocks J solved so far (gathered in Xg, ld n_loc)
  for (int K = 0; K < d.nblk; ++K) {
    const int orow = K % d.r, ocol = K % d.c, owner = orow * d.c + ocol;
    double* XK = X + (long long)K * nb;
    if (d.pr == orow) {
      if (ng > 0)
        GG_TRY(local_gemm(nb, k, ng * nb, 1.0, L + d.lrow(K), lda, w.Xg, d.n_loc, false, 0.0,
                          w.part, nb, nullptr, 0, s));
      else
        GG_CUDA_TRY(cudaMemsetAsync(w.part, 0, (size_t)nb * k * 8, s));
      GG_TRY(coll_sum(cm, G_ROW, w.part, (size_t)nb * k, s));
      if (cm->rank == owner) {
        GG_CUDA_TRY(cudaMemcpy2DAsync(w.Lkk, (size_t)nb * 8, L + d.lrow(K) + d.lcol(K) * lda,
                                      lda * 8, (size_t)nb * 8, nb, cudaMemcpyDeviceToDevice, s));
        GG_TRY(trtri_run(nb, w.Lkk, nb, w.Dinv, nb, w.tws, s));
        sub_block_kernel<<<64, 256, 0, s>>>(nb, k, XK, ldx, w.part, nb, w.rhs);
        GG_LAUNCH_CHECK("sub_block_kernel");
        GG_TRY(local_gemm(nb, k, nb, 1.0, w.Dinv, nb, w.rhs, nb, false, 0.0, w.xk, nb, nullptr, 0,
                          s));
      }
    }
    GG_TRY(coll_bcast(cm, G_WORLD, w.xk, (size_t)nb * k * 8, owner, s));
    GG_CUDA_TRY(cudaMemcpy2DAsync(XK, ldx * 8, w.xk, (size_t)nb * 8, (size_t)nb * 8, k,
                                  cudaMemcpyDeviceToDevice, s));
    if (K % d.c == d.pc) {   // one of this rank's column blocks: keep its rows for later products
      GG_CUDA_TRY(cudaMemcpy2DAsync(w.Xg + (long long)ng * nb, (size_t)d.n_loc * 8, w.xk,
                                    (size_t)nb * 8, (size_t)nb * 8, k, cudaMemcpyDeviceToDevice, s));
      ++ng;
    }
  }
  return GG_OK;
}

}  // namespace
}  // namespace gg

extern "C" {

int gg_dist_nccl_unique_id(unsigned char* id_out) {
  if (id_out == nullptr) {
    gg::set_error("dist: null id buffer");
    return GG_EARG;
  }
  const gg::NcclApi& a = gg::nccl();
  if (!a.ok) {
    gg::set_error("dist: libnccl.so.2 not available in this process");
    return GG_ENCCL;
  }
  ncclUniqueId id;
  GG_NCCL_TRY(a.getUniqueId(&id), "ncclGetUniqueId");
  memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return GG_OK;
}

static int comms_check(int rank, int nranks, int grid_r, int grid_c) {
  if (nranks < 1 || rank < 0 || rank >= nranks || grid_r < 1 || grid_c < 1 ||
      grid_r * grid_c != nranks) {
    gg::set_error("dist: rank / grid inconsistent (grid_r * grid_c must equal nranks)");
    return GG_EARG;
  }
  return GG_OK;
}

int gg_dist_comms_nccl(int rank, int nranks, int grid_r, int grid_c, const unsigned char* id,
                       gg_dist_comms** out) {
  GG_NVTX("gg_dist_comms_nccl");
  if (out == nullptr || id == nullptr) {
    gg::set_error("dist: null argument");
    return GG_EARG;
  }
  *out = nullptr;
  int rc = comms_check(rank, nranks, grid_r, grid_c);
  if (rc != GG_OK) return rc;
  const gg::NcclApi& a = gg::nccl();
  if (!a.ok) {
    gg::set_error("dist: libnccl.so.2 not available in this process");
    return GG_ENCCL;
  }
  auto* c = new gg_dist_comms{};
  c->rank = rank; c->nranks = nranks; c->r = grid_r; c->c = grid_c;
  c->pr = rank / grid_c; c->pc = rank % grid_c;
  c->use_nccl = true;
  ncclUniqueId uid;
  memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclResult_t r = a.commInitRank(&c->comm[gg::G_WORLD], nranks, uid, rank);
  if (r == ncclSuccess)   // process row (key = column index) and process column (key = row index)
    r = a.commSplit(c->comm[gg::G_WORLD], c->pr, c->pc, &c->comm[gg::G_ROW], nullptr);
  if (r == ncclSuccess)
    r = a.commSplit(c->comm[gg::G_WORLD], grid_r + c->pc, c->pr, &c->comm[gg::G_COL], nullptr);
  if (r != ncclSuccess) {
    gg_dist_comms_free(c);
    return gg::nccl_fail(r, "NCCL communicator setup");
  }
  *out = c;
  return GG_OK;
}

int gg_dist_comms_callbacks(int rank, int nranks, int grid_r, int grid_c, gg_dist_bcast_fn bcast,
                            gg_dist_allreduce_fn allreduce, void* ctx, gg_dist_comms** out) {
  if (out == nullptr || (nranks > 1 && (bcast == nullptr || allreduce == nullptr))) {
    gg::set_error("dist: null argument");
    return GG_EARG;
  }
  *out = nullptr;
  int rc = comms_check(rank, nranks, grid_r, grid_c);
  if (rc != GG_OK) return rc;
  auto* c = new gg_dist_comms{};
  c->rank = rank; c->nranks = nranks; c->r = grid_r; c->c = grid_c;
  c->pr = rank / grid_c; c->pc = rank % grid_c;
  c->use_nccl = false;
  c->bcast = bcast; c->allreduce = allreduce; c->ctx = ctx;
  *out = c;
  return GG_OK;
}

int gg_dist_comms_free(gg_dist_comms* c) {
  if (c == nullptr) return GG_OK;
  if (c->use_nccl) {
    const gg::NcclApi& a = gg::nccl();
    for (int g = 2; g >= 0; --g)
      if (c->comm[g] != nullptr && a.commDestroy) a.commDestroy(c->comm[g]);
  }
  delete c;
  return GG_OK;
}

int gg_dist_local_dims(int n, int nb, const gg_dist_comms* c, int* m_loc, int* n_loc) {
  if (c == nullptr || m_loc == nullptr || n_loc == nullptr || n < 1 || nb < 1) {
    gg::set_error("dist: null argument or bad size");
    return GG_EARG;
  }
  const gg::DistShape d(n, nb, c);
  *m_loc = d.m_loc;
  *n_loc = d.n_loc;
  return GG_OK;
}

size_t gg_dist_potrf_workspace_bytes(int n, int nb, const gg_dist_comms* c) {
  if (c == nullptr || n < 1 || nb < 1) return 0;
  const gg::DistShape d(n, nb, c);
  return gg::DistWork(d, nullptr).total;
}

int gg_dist_potrf_f64(int n, int nb, double* A, long long lda, double* B, long long ldb,
                      const gg_dist_comms* c, void* work, size_t work_bytes, int* info,
                      void* stream) {
  GG_NVTX("gg_dist_potrf_f64");
  if (c == nullptr || work == nullptr || info == nullptr || n < 1 || nb < GG_TILE ||
      nb % GG_TILE != 0) {
    gg::set_error("dist_potrf: null pointer, n < 1, or nb not a positive multiple of 128");
    return GG_EARG;
  }
  const gg::DistShape d(n, nb, c);
  if ((A == nullptr || B == nullptr) && (long long)d.m_loc * d.n_loc > 0) {   // empty shares: any
    gg::set_error("dist_potrf: null local share");
    return GG_EARG;
  }
  *info = -1;
  return gg::dist_potrf_run(n, nb, A, lda, B, ldb, c, work, work_bytes, info,
                            static_cast<cudaStream_t>(stream));
}

size_t gg_dist_trsm_workspace_bytes(int n, int nb, int nrhs, const gg_dist_comms* c) {
  if (c == nullptr || n < 1 || nb < 1) return 0;
  const gg::DistShape d(n, nb, c);
  return gg::TrsmWork(d, nrhs, nullptr).total;
}

int gg_dist_trsm_f64(int n, int nb, int nrhs, const double* L, long long lda, double* X,
                     long long ldx, const gg_dist_comms* c, void* work, size_t work_bytes,
                     void* stream) {
  GG_NVTX("gg_dist_trsm_f64");
  if (c == nullptr || X == nullptr || work == nullptr || n < 1 || nrhs < 0 || nb < GG_TILE ||
      nb % GG_TILE != 0) {
    gg::set_error("dist_trsm: null pointer, bad size, or nb not a positive multiple of 128");
    return GG_EARG;
  }
  const gg::DistShape d(n, nb, c);
  if (L == nullptr && (long long)d.m_loc * d.n_loc > 0) {
    gg::set_error("dist_trsm: null local share");
    return GG_EARG;
  }
  return gg::dist_trsm_run(n, nb, nrhs, L, lda, X, ldx, c, work, work_bytes,
                           static_cast<cudaStream_t>(stream));
}

}  // extern "C"
