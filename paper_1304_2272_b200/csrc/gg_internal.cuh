// Internal declarations shared by the sm_100a translation units of libgwasgls_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/gwasgls_b200.h"

namespace gg {

// ---- error plumbing (thread-local message, no global mutable state) -----------------
void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define GG_CUDA_TRY(expr)                                                   \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) return ::gg::cuda_fail(_e, #expr);               \
  } while (0)

#define GG_LAUNCH_CHECK(what)                                               \
  do {                                                                      \
    cudaError_t _e = cudaGetLastError();                                    \
    if (_e != cudaSuccess) return ::gg::cuda_fail(_e, what);                \
  } while (0)

#define GG_TRY(expr)                                                        \
  do {                                                                      \
    const int _rc = (expr);                                                 \
    if (_rc != GG_OK) return _rc;                                           \
  } while (0)

inline int pad_rows(int n) { return ((n + GG_TILE - 1) / GG_TILE) * GG_TILE; }

// NVTX range around a C-ABI entry point (header-only NVTX 3: a few ns when no tool listens);
// nsys / ncu --nvtx see gg_* ranges around every library call.
struct NvtxRange {
  explicit NvtxRange(const char* name);
  ~NvtxRange();
};
#define GG_NVTX(name) ::gg::NvtxRange _gg_nvtx_range(name)

// ---- FP64 DMMA GEMM (gemm_f64.cu) ----------------------------------------------------
enum GemmFlags : int {
  GEMM_A_LOWER = 1,   // A lower triangular: row tile mt only needs k < (mt+1)*BM
  GEMM_B_LOWER = 2,   // op(B) lower triangular (k >= n): column tile nt needs k >= nt*BN
  GEMM_C_LOWER = 4,   // only tiles on/below the diagonal are computed (SYRK; C's origin on
                      // the diagonal, N <= M)
};

struct GemmArgs {
  int M, N, K;        // M % 128 == 0, K % 16 == 0, N >= 1 arbitrary
  const double* A;  long long lda;
  const double* B;  long long ldb;
  double* C;        long long ldc;
  double alpha, beta;
  int flags;
  const int* abort_flag;   // optional device flag: kernel is a no-op when *abort_flag != 0
  int batch;                // strided batch (0 or 1: one problem): problem z uses
  long long sA, sB, sC;     // A + z sA, B + z sB, C + z sC (same shape and flags)
};

// Launch C = alpha*A*op(B) + beta*C.  trans_b selects op(B) = B^T (B stored N x K).
int launch_dgemm(const GemmArgs& a, bool trans_b, cudaStream_t s);

// ---- FP64 GEMM on the int8 tensor cores, Ozaki scheme (ozaki_i8.cu) -------------------------
// C = beta C + alpha A~ B~^T, A~(i,k) = A[i a_rs + k a_cs] (M x K), B~(j,k) = B[j b_rs + k b_cs]
// (N x K; B == nullptr: B~ = A~).  flags: GEMM_A_LOWER (A~(i,k) = 0 for k > i), GEMM_B_LOWER
// (B~(j,k) = 0 for k < j), GEMM_C_LOWER (tiles strictly above the diagonal skipped).
size_t ozaki_ws_bytes(int M, int N, int K, bool b_is_a);
int ozaki_gemm_run(int M, int N, int K, const double* A, long long a_rs, long long a_cs,
                   const double* B, long long b_rs, long long b_cs, double* C, long long ldc,
                   double alpha, double beta, int flags, void* ws, size_t ws_bytes,
                   const int* abort_flag, cudaStream_t s);

// ---- dense factorisation (potrf_f64.cu) ----------------------------------------------
int potrf_run(int n, const double* M, int ldm, int m_row_major, double* L, double* Linv, int ldp,
              void* work,
              int* info_host, cudaStream_t s);
int trtri_run(int n, const double* L, int ldl, double* Linv, int ldp, void* work,
              cudaStream_t s);
size_t potrf_ws_bytes(int n);
size_t trtri_ws_bytes(int n);
size_t trsm_blocked_ws_bytes(int n, int nrhs);
int trsm_blocked_run(int n, int nrhs, const double* L, int ldl, const double* B, int ldb,
                     double* X, int ldx, void* work, cudaStream_t s);

// ---- TMA/DMMA streamed TRSM (trsm_tma.cu) -------------------------------------------------
int trsm_rowmajor_run(int n, int nrhs, const double* LinvT, int ldp, const double* B, int ldb,
                      double* X, int ldx, cudaStream_t s);
int trsm_packed_run(int n, int nrhs, const double* LinvP, const double* B, int ldb, double* X,
                    int ldx, cudaStream_t s);
int trsm_packed_gated_run(int n, int nrhs, const double* LinvP, const double* B, int ldb,
                          double* X, int ldx, const int* gate, int gate_value, cudaStream_t s);
size_t packed_lower_elems(int n);
int pack_lower_run(int n, const double* A, int lda, int row_major, double* P, cudaStream_t s);
int pack_lower_bc_run(int n, int nb, int gr, int gc, int pr, int pc, const double* B, int ldl,
                      double* P, cudaStream_t s);
int transpose_square_run(int np, const double* A, int lda, double* T, int ldt, cudaStream_t s);

// ---- int8 tensor-core TRSM with the sliced inverse (trsm_i8.cu) -----------------------------
int i8_slices();
size_t inverse_slices_bytes(int n);
int slice_inverse_run(int n, const double* LinvT, int ldp, signed char* Sl, int* expo,
                      cudaStream_t s);
int i8_value_bound(int n);
int slice_packed_run(int n, const double* LinvP, signed char* Sl, int* meta, cudaStream_t s);
size_t slice_meta_ints(int n);
int row_exponents_bc_run(int n, int nb, int gr, int gc, int pr, int pc, const double* B, int ldl,
                         int* ex2, cudaStream_t s);
int slice_meta_run(int n, const int* ex2, int* meta, cudaStream_t s);
int slice_bc_run(int n, int nb, int gr, int gc, int pr, int pc, const double* B, int ldl,
                 int* meta, signed char* Sl, cudaStream_t s);
// per-column flags (colbad, cnt ints, nullable; set to 1 for a flagged column, never cleared)
// plus a block flag (*bad |= 1 if any column is flagged)
int range_i8_run(int n, int cnt, const signed char* G, long long ldg, int* bad, int* colbad,
                 cudaStream_t s);
int narrow_run(int n, int cnt, const double* X, long long ldx, signed char* G, long long ldg,
               int* bad, int* colbad, cudaStream_t s);
// counter: one device int of the caller's workspace (the dynamic tile scheduler)
int trsm_i8_run(int n, int nrhs, const signed char* Sl, const int* expo, const signed char* G,
                long long ldg, double* X, int ldx, int* counter, cudaStream_t s);
int trsm_i8_fused_run(int n, int nrhs, const signed char* Sl, const int* expo,
                      const signed char* G, long long ldg, double* X, int ldx, int q,
                      const double* XL, int ldxl, const double* y, double* P, const int* gate,
                      int gate_value, int* counter, cudaStream_t s);

// ---- GLS epilogue + helpers (gls_epilogue.cu) ----------------------------------------
int dots_run(int n, int cnt, int q, const double* Xbar, int ldx, const double* XLbar,
             int ldxl, const double* ybar, double* dots, double* P, cudaStream_t s);
int small_solve_run(int batch, int p, const double* S, const double* rhs, double* x,
                    int* status, double* sinv, cudaStream_t s);
int epilogue_run(int n, int cnt, int q, const double* Xbar, int ldx, const double* XLbar,
                 int ldxl, const double* ybar, const double* S_TL, const double* b_T,
                 double* beta, int* status, double* sinv, double* P, cudaStream_t s);
int widen_run(int n, int cnt, const int8_t* G, long long ldg, double* X, int ldx,
              cudaStream_t s);
size_t partials_bytes(int n, int cnt, int q);
// colmask (nullable): only columns with colmask[j] != 0 are written
int partials_run(int n, int cnt, int q, const double* Xbar, int ldx, const double* XLbar,
                 int ldxl, const double* ybar, double* P, cudaStream_t s, const int* gate,
                 int gate_value, const int* colmask = nullptr);
int mark_invalid_run(int cnt, int p, const int* gate, int gate_value, double* beta, int* status,
                     cudaStream_t s, const int* colmask = nullptr);
int reduce_solve_run(int n, int cnt, int q, const double* P, double* dots, const double* S_TL,
                     const double* b_T, double* beta, int* status, double* sinv, cudaStream_t s);

// ---- generator (datagen.cu) -----------------------------------------------------------
int gen_genotypes_run(unsigned long long seed, int stream_maf, int stream_geno, int n,
                      long long m, long long first, int cnt, double maf_lo, double maf_hi,
                      int8_t* G, long long ldg, double* Z, int ldz, cudaStream_t s);

}  // namespace gg
