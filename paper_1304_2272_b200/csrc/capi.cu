// extern "C" entry points of libgwasgls_b200.so (declared in include/gwasgls_b200.h).
// Each validates its arguments, runs on the caller's stream and current device, and reports
// failures through a status code plus a thread-local message.
#include <nvtx3/nvToolsExt.h>

#include <cstdio>
#include <string>

#include "gg_internal.cuh"

namespace gg {

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return GG_ECUDA;
}

}  // namespace gg

using gg::pad_rows;

static inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }
static inline const signed char* slices_as(const int8_t* p) {
  return reinterpret_cast<const signed char*>(p);
}

extern "C" {

const char* gg_version(void) { return "gwasgls_b200 0.1.0 (sm_100a, FP64 DMMA)"; }

const char* gg_last_error(void) { return gg::g_last_error.c_str(); }

int gg_pad(int n) { return pad_rows(n); }

size_t gg_potrf_workspace_bytes(int n) { return n < 1 ? 0 : gg::potrf_ws_bytes(n); }

int gg_potrf_f64(int n, const double* M, int ldm, int m_row_major, double* L, double* Linv,
                 int ldp, void* work, int* info_host, void* stream) {
  GG_NVTX("gg_potrf_f64");
  return gg::potrf_run(n, M, ldm, m_row_major, L, Linv, ldp, work, info_host, as_stream(stream));
}

size_t gg_trtri_workspace_bytes(int n) { return n < 1 ? 0 : gg::trtri_ws_bytes(n); }

int gg_trtri_lower_f64(int n, const double* L, int ldl, double* Linv, int ldp, void* work,
                       void* stream) {
  GG_NVTX("gg_trtri_lower_f64");
  return gg::trtri_run(n, L, ldl, Linv, ldp, work, as_stream(stream));
}

size_t gg_trsm_lower_blocked_workspace_bytes(int n, int nrhs) {
  return n < 1 ? 0 : gg::trsm_blocked_ws_bytes(n, nrhs);
}

int gg_trsm_lower_blocked_f64(int n, int nrhs, const double* L, int ldl, const double* B,
                              int ldb, double* X, int ldx, void* work, void* stream) {
  GG_NVTX("gg_trsm_lower_blocked_f64");
  if (n < 1 || nrhs < 0 || L == nullptr || B == nullptr || X == nullptr || work == nullptr) {
    gg::set_error("trsm_blocked: null pointer or bad size");
    return GG_EARG;
  }
  return gg::trsm_blocked_run(n, nrhs, L, ldl, B, ldb, X, ldx, work, as_stream(stream));
}

int gg_trsm_lower_f64(int n, int nrhs, const double* Linv, int ldp, const double* B, int ldb,
                      double* X, int ldx, void* stream) {
  if (n < 1 || nrhs < 0 || Linv == nullptr || B == nullptr || X == nullptr) {
    gg::set_error("trsm: null pointer or bad size");
    return GG_EARG;
  }
  if (B == X) {
    gg::set_error("trsm: X must not alias B");
    return GG_EARG;
  }
  const int np = pad_rows(n);
  if (ldp < np || ldb < np || ldx < np) {
    gg::set_error("trsm: leading dimensions must be >= gg_pad(n)");
    return GG_EDIM;
  }
  if (nrhs == 0) return GG_OK;
  gg::GemmArgs a{};
  a.M = np; a.N = nrhs; a.K = np;
  a.A = Linv; a.lda = ldp;
  a.B = B; a.ldb = ldb;
  a.C = X; a.ldc = ldx;
  a.alpha = 1.0; a.beta = 0.0;
  a.flags = gg::GEMM_A_LOWER;
  a.abort_flag = nullptr;
  return gg::launch_dgemm(a, false, as_stream(stream));
}

int gg_trsm_lower_rm_f64(int n, int nrhs, const double* LinvT, int ldp, const double* B,
                         int ldb, double* X, int ldx, void* stream) {
  if (n < 1 || nrhs < 0 || LinvT == nullptr || B == nullptr || X == nullptr) {
    gg::set_error("trsm: null pointer or bad size");
    return GG_EARG;
  }
  if (B == X) {
    gg::set_error("trsm: X must not alias B");
    return GG_EARG;
  }
  return gg::trsm_rowmajor_run(n, nrhs, LinvT, ldp, B, ldb, X, ldx, as_stream(stream));
}

size_t gg_packed_lower_bytes(int n) {
  return n < 1 ? 0 : gg::packed_lower_elems(n) * sizeof(double);
}

int gg_pack_lower_f64(int n, const double* A, int lda, int row_major, double* LinvP,
                      void* stream) {
  if (n < 1 || A == nullptr || LinvP == nullptr) {
    gg::set_error("pack_lower: null pointer or n < 1");
    return GG_EARG;
  }
  return gg::pack_lower_run(n, A, lda, row_major, LinvP, as_stream(stream));
}

int gg_pack_lower_blockcyclic_f64(int n, int nb, int grid_r, int grid_c, int prow, int pcol,
                                  const double* Bloc, int ldloc, double* LinvP, void* stream) {
  if (n < 1 || Bloc == nullptr || LinvP == nullptr) {
    gg::set_error("pack_lower_blockcyclic: null pointer or n < 1");
    return GG_EARG;
  }
  return gg::pack_lower_bc_run(n, nb, grid_r, grid_c, prow, pcol, Bloc, ldloc, LinvP,
                               as_stream(stream));
}

int gg_trsm_lower_packed_f64(int n, int nrhs, const double* LinvP, const double* B, int ldb,
                             double* X, int ldx, void* stream) {
  GG_NVTX("gg_trsm_lower_packed_f64");
  if (n < 1 || nrhs < 0 || LinvP == nullptr || B == nullptr || X == nullptr) {
    gg::set_error("trsm: null pointer or bad size");
    return GG_EARG;
  }
  if (B == X) {
    gg::set_error("trsm: X must not alias B");
    return GG_EARG;
  }
  return gg::trsm_packed_run(n, nrhs, LinvP, B, ldb, X, ldx, as_stream(stream));
}

int gg_i8_slices(void) { return gg::i8_slices(); }

int gg_i8_value_bound(int n) { return gg::i8_value_bound(n); }

size_t gg_inverse_slices_bytes(int n) { return n < 1 ? 0 : gg::inverse_slices_bytes(n); }

int gg_slice_inverse_i8(int n, const double* LinvT, int ldp, int8_t* slices, int* expo,
                        void* stream) {
  GG_NVTX("gg_slice_inverse_i8");
  if (n < 1 || LinvT == nullptr || slices == nullptr || expo == nullptr) {
    gg::set_error("slice_inverse: null pointer or n < 1");
    return GG_EARG;
  }
  return gg::slice_inverse_run(n, LinvT, ldp, reinterpret_cast<signed char*>(slices), expo,
                               as_stream(stream));
}

int gg_slice_packed_inverse_i8(int n, const double* LinvP, int8_t* slices, int* expo,
                               void* stream) {
  GG_NVTX("gg_slice_packed_inverse_i8");
  if (n < 1 || LinvP == nullptr || slices == nullptr || expo == nullptr) {
    gg::set_error("slice_packed_inverse: null pointer or n < 1");
    return GG_EARG;
  }
  return gg::slice_packed_run(n, LinvP, reinterpret_cast<signed char*>(slices), expo,
                              as_stream(stream));
}

size_t gg_slice_meta_ints(int n) { return n < 1 ? 0 : gg::slice_meta_ints(n); }

int gg_row_exponents_blockcyclic(int n, int nb, int grid_r, int grid_c, int prow, int pcol,
                                 const double* Bloc, int ldloc, int* ex2, void* stream) {
  if (n < 1 || Bloc == nullptr || ex2 == nullptr) {
    gg::set_error("row_exponents_blockcyclic: null pointer or n < 1");
    return GG_EARG;
  }
  return gg::row_exponents_bc_run(n, nb, grid_r, grid_c, prow, pcol, Bloc, ldloc, ex2,
                                  as_stream(stream));
}

int gg_slice_meta_i8(int n, const int* ex2, int* expo, void* stream) {
  if (n < 1 || ex2 == nullptr || expo == nullptr) {
    gg::set_error("slice_meta: null pointer or n < 1");
    return GG_EARG;
  }
  return gg::slice_meta_run(n, ex2, expo, as_stream(stream));
}

int gg_slice_blockcyclic_i8(int n, int nb, int grid_r, int grid_c, int prow, int pcol,
                            const double* Bloc, int ldloc, int* expo, int8_t* slices,
                            void* stream) {
  if (n < 1 || Bloc == nullptr || expo == nullptr || slices == nullptr) {
    gg::set_error("slice_blockcyclic: null pointer or n < 1");
    return GG_EARG;
  }
  return gg::slice_bc_run(n, nb, grid_r, grid_c, prow, pcol, Bloc, ldloc, expo,
                          reinterpret_cast<signed char*>(slices), as_stream(stream));
}

int gg_narrow_f64_i8(int n, int cnt, const double* X, long long ldx, int8_t* G, long long ldg,
                     int* bad_dev, void* stream) {
  GG_NVTX("gg_narrow_f64_i8");
  if (n < 1 || X == nullptr || G == nullptr || bad_dev == nullptr) {
    gg::set_error("narrow: null pointer or n < 1");
    return GG_EARG;
  }
  return gg::narrow_run(n, cnt, X, ldx, reinterpret_cast<signed char*>(G), ldg, bad_dev, nullptr,
                        as_stream(stream));
}

size_t gg_trsm_i8_workspace_bytes(void) { return 256; }

int gg_trsm_lower_i8(int n, int nrhs, const int8_t* slices, const int* expo, const int8_t* G,
                     long long ldg, double* X, int ldx, void* work, void* stream) {
  GG_NVTX("gg_trsm_lower_i8");
  if (n < 1 || nrhs < 0 || slices == nullptr || expo == nullptr || G == nullptr || X == nullptr ||
      work == nullptr) {
    gg::set_error("trsm_i8: null pointer or bad size");
    return GG_EARG;
  }
  return gg::trsm_i8_run(n, nrhs, reinterpret_cast<const signed char*>(slices), expo,
                         reinterpret_cast<const signed char*>(G), ldg, X, ldx,
                         static_cast<int*>(work), as_stream(stream));
}

size_t gg_partials_bytes(int n, int cnt, int q) {
  return (n < 1 || cnt < 1 || q < 0) ? 0 : gg::partials_bytes(n, cnt, q);
}

int gg_trsm_lower_i8_partials(int n, int cnt, const int8_t* slices, const int* expo,
                              const int8_t* G, long long ldg, int q, const double* XLbar,
                              const double* ybar, double* P, double* X, int ldx, const int* gate,
                              int gate_value, void* work, void* stream) {
  GG_NVTX("gg_trsm_lower_i8_partials");
  if (n < 1 || cnt < 0 || slices == nullptr || expo == nullptr || G == nullptr || P == nullptr ||
      ybar == nullptr || (q > 0 && XLbar == nullptr) || q < 0 || q > GG_PMAX - 1 ||
      work == nullptr) {
    gg::set_error("trsm_i8_partials: null pointer or bad size");
    return GG_EARG;
  }
  return gg::trsm_i8_fused_run(n, cnt, slices_as(slices), expo,
                               reinterpret_cast<const signed char*>(G), ldg, X, ldx, q, XLbar,
                               pad_rows(n), ybar, P, gate, gate_value, static_cast<int*>(work),
                               as_stream(stream));
}

int gg_gls_reduce_solve_f64(int n, int cnt, int q, const double* P, const double* S_TL,
                            const double* b_T, double* beta, int* status, double* sinv,
                            void* stream) {
  GG_NVTX("gg_gls_reduce_solve_f64");
  if (n < 1 || P == nullptr || beta == nullptr || status == nullptr || q < 0 || q > GG_PMAX - 1 ||
      (q > 0 && (S_TL == nullptr || b_T == nullptr))) {
    gg::set_error("reduce_solve: null pointer or bad size");
    return GG_EARG;
  }
  if (cnt <= 0) return GG_OK;
  return gg::reduce_solve_run(n, cnt, q, P, nullptr, S_TL, b_T, beta, status, sinv,
                              as_stream(stream));
}

int gg_transpose_f64(int np, const double* A, int lda, double* T, int ldt, void* stream) {
  if (A == nullptr || T == nullptr || A == T) {
    gg::set_error("transpose: null or aliased pointers");
    return GG_EARG;
  }
  return gg::transpose_square_run(np, A, lda, T, ldt, as_stream(stream));
}

size_t gg_gemm_ozaki_workspace_bytes(int m, int ncols, int k, int b_is_a) {
  if (m < 1 || ncols < 1 || k < 1) return 0;
  return gg::ozaki_ws_bytes(m, ncols, k, b_is_a != 0);
}

int gg_gemm_ozaki_f64(int m, int ncols, int k, const double* A, long long a_rs, long long a_cs,
                      const double* B, long long b_rs, long long b_cs, double* C, long long ldc,
                      double alpha, double beta, int flags, void* work, size_t work_bytes,
                      void* stream) {
  GG_NVTX("gg_gemm_ozaki_f64");
  if (A == nullptr || C == nullptr || m < 0 || ncols < 0 || k < 0 || ldc < m ||
      (flags & ~7) != 0) {
    gg::set_error("gemm_ozaki: bad arguments");
    return GG_EARG;
  }
  return gg::ozaki_gemm_run(m, ncols, k, A, a_rs, a_cs, B, b_rs, b_cs, C, ldc, alpha, beta, flags,
                            work, work_bytes, nullptr, as_stream(stream));
}

int gg_dgemm_f64(int m, int ncols, int k, double alpha, const double* A, int lda, const double* B,
                 int ldb, int trans_b, double beta, double* C, int ldc, void* stream) {
  if (A == nullptr || B == nullptr || C == nullptr) {
    gg::set_error("dgemm: null pointer");
    return GG_EARG;
  }
  gg::GemmArgs a{};
  a.M = m; a.N = ncols; a.K = k;
  a.A = A; a.lda = lda;
  a.B = B; a.ldb = ldb;
  a.C = C; a.ldc = ldc;
  a.alpha = alpha; a.beta = beta;
  a.flags = 0;
  a.abort_flag = nullptr;
  return gg::launch_dgemm(a, trans_b != 0, as_stream(stream));
}

int gg_widen_i8_f64(int n, int cnt, const int8_t* G, long long ldg, double* X, int ldx,
                    void* stream) {
  if (n < 1 || cnt < 0 || G == nullptr || X == nullptr) {
    gg::set_error("widen: null pointer or bad size");
    return GG_EARG;
  }
  return gg::widen_run(n, cnt, G, ldg, X, ldx, as_stream(stream));
}

int gg_gls_dots_f64(int n, int cnt, int q, const double* Xbar, int ldx, const double* XLbar,
                    int ldxl, const double* ybar, double* dots, void* work, void* stream) {
  GG_NVTX("gg_gls_dots_f64");
  if (Xbar == nullptr || ybar == nullptr || dots == nullptr || work == nullptr ||
      (q > 0 && XLbar == nullptr)) {
    gg::set_error("dots: null pointer");
    return GG_EARG;
  }
  return gg::dots_run(n, cnt, q, Xbar, ldx, XLbar, ldxl, ybar, dots,
                      static_cast<double*>(work), as_stream(stream));
}

int gg_small_spd_solve_f64(int batch, int p, const double* S, const double* rhs, double* x,
                           int* status, double* sinv_packed, void* stream) {
  GG_NVTX("gg_small_spd_solve_f64");
  if (S == nullptr || rhs == nullptr || x == nullptr || status == nullptr) {
    gg::set_error("small_spd_solve: null pointer");
    return GG_EARG;
  }
  return gg::small_solve_run(batch, p, S, rhs, x, status, sinv_packed, as_stream(stream));
}

int gg_gls_epilogue_f64(int n, int cnt, int q, const double* Xbar, int ldx, const double* XLbar,
                        int ldxl, const double* ybar, const double* S_TL, const double* b_T,
                        double* beta, int* status, double* sinv, void* work, void* stream) {
  GG_NVTX("gg_gls_epilogue_f64");
  if (Xbar == nullptr || ybar == nullptr || beta == nullptr || status == nullptr ||
      work == nullptr || (q > 0 && (XLbar == nullptr || S_TL == nullptr || b_T == nullptr))) {
    gg::set_error("epilogue: null pointer");
    return GG_EARG;
  }
  return gg::epilogue_run(n, cnt, q, Xbar, ldx, XLbar, ldxl, ybar, S_TL, b_T, beta, status, sinv,
                          static_cast<double*>(work), as_stream(stream));
}

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct BlockWs {
  int* flag;      // block flag: some column takes the FP64 path
  int* counter;   // tile counter of the int8 TRSM's dynamic scheduler
  int* colbad;    // per-column flags (cnt ints): 1 = this column takes the FP64 path
  double* P;
  signed char* g8;
  double* x64;
  double* xbar;
  size_t bytes;
};

// Workspace layout of gg_gls_block_f64 (what each input kind / path needs).
static BlockWs block_ws(int n, int q, int cnt, int input_int8, int have_slices, char* base) {
  const size_t np = (size_t)pad_rows(n), n16 = (size_t)((n + 15) / 16 * 16);
  BlockWs w{};
  size_t off = 256;   // flag at 0, tile counter at 128
  w.flag = reinterpret_cast<int*>(base);
  w.counter = reinterpret_cast<int*>(base + 128);
  w.colbad = reinterpret_cast<int*>(base + off);
  off += align256(sizeof(int) * (size_t)cnt);
  w.P = reinterpret_cast<double*>(base + off);
  off += align256(gg::partials_bytes(n, cnt, q));
  // int8 input at n > 132,104: values beyond gg_i8_value_bound(n) take the DMMA path
  const bool i8_guard = have_slices && input_int8 && gg::i8_value_bound(n) < 127;
  const bool need_g8 = have_slices;                              // narrowed / re-pitched dosages
  const bool need_x64 = (!have_slices && input_int8) || i8_guard;   // widened dosages (DMMA)
  const bool need_xbar = !(have_slices && input_int8) || i8_guard;  // DMMA result
  w.g8 = need_g8 ? reinterpret_cast<signed char*>(base + off) : nullptr;
  if (need_g8) off += align256(n16 * cnt);
  w.x64 = need_x64 ? reinterpret_cast<double*>(base + off) : nullptr;
  if (need_x64) off += align256(np * cnt * sizeof(double));
  w.xbar = need_xbar ? reinterpret_cast<double*>(base + off) : nullptr;
  if (need_xbar) off += align256(np * cnt * sizeof(double));
  w.bytes = off;
  return w;
}

size_t gg_gls_block_workspace_bytes(int n, int q, int cnt, int input_int8, int have_slices) {
  if (n < 1 || cnt < 1) return 256;
  return block_ws(n, q, cnt, input_int8, have_slices, nullptr).bytes;
}

int gg_gls_block_f64(int n, int q, int cnt, const double* LinvP, const int8_t* slices,
                     const int* expo, const double* XLbar, const double* ybar, const double* S_TL,
                     const double* b_T, const double* X64, int ldx, const int8_t* G8,
                     long long ldg, void* work, double* beta, int* status, double* sinv,
                     void* stream) {
  GG_NVTX("gg_gls_block_f64");
  cudaStream_t s = as_stream(stream);
  if ((X64 == nullptr) == (G8 == nullptr)) {
    gg::set_error("gls_block: exactly one of X64 / G8 must be given");
    return GG_EARG;
  }
  const bool have_slices = slices != nullptr && expo != nullptr;
  if (work == nullptr || (LinvP == nullptr && !have_slices)) {
    gg::set_error("gls_block: null workspace / inverse");
    return GG_EARG;
  }
  if (q < 0 || q > GG_PMAX - 1) {
    gg::set_error("gls_block: need 0 <= q <= 19");
    return GG_EARG;
  }
  if (cnt <= 0) return GG_OK;
  const int np = pad_rows(n);
  const long long n16 = (n + 15) / 16 * 16;
  const BlockWs w = block_ws(n, q, cnt, G8 != nullptr, have_slices, static_cast<char*>(work));
  int rc = GG_OK;
  bool invalid_gate = false;
  if (have_slices) {
    // Per-column path selection, on the device (no host sync): a column whose values the int8
    // tensor-core path cannot compute exactly (non-integer, or beyond gg_i8_value_bound(n)) is
    // flagged on its own; the int8 TRSM runs for the whole block, then -- only if some column is
    // flagged -- the FP64 DMMA TRSM and the reductions overwrite the flagged columns' partials.
    // A column's path, and so its result, depends only on its own values.
    GG_CUDA_TRY(cudaMemsetAsync(w.flag, 0, sizeof(int), s));
    GG_CUDA_TRY(cudaMemsetAsync(w.colbad, 0, sizeof(int) * (size_t)cnt, s));
    const signed char* g = reinterpret_cast<const signed char*>(G8);
    long long lg = ldg;
    const double* x64 = X64;   // FP64 columns for the DMMA path
    int ldx64 = ldx;
    bool may_flag = true;
    if (G8 != nullptr) {
      if (ldg % 16 != 0 || (reinterpret_cast<uintptr_t>(G8) & 15)) {   // re-pitch for TMA
        GG_CUDA_TRY(cudaMemcpy2DAsync(w.g8, n16, G8, ldg, n, cnt, cudaMemcpyDeviceToDevice, s));
        g = w.g8;
        lg = n16;
      }
      // large n only: values beyond the exact-int32 bound take the FP64 path
      may_flag = gg::i8_value_bound(n) < 127;
      if (may_flag) rc = gg::range_i8_run(n, cnt, g, lg, w.flag, w.colbad, s);
    } else {
      rc = gg::narrow_run(n, cnt, X64, ldx, w.g8, n16, w.flag, w.colbad, s);
      g = w.g8;
      lg = n16;
    }
    if (rc == GG_OK)
      rc = gg::trsm_i8_fused_run(n, cnt, slices_as(slices), expo, g, lg, nullptr, 0, q, XLbar,
                                 np, ybar, w.P, nullptr, 0, w.counter, s);
    if (rc == GG_OK && may_flag && LinvP != nullptr) {
      if (G8 != nullptr) {
        rc = gg::widen_run(n, cnt, G8, ldg, w.x64, np, s);   // (a no-op grid when unflagged
        x64 = w.x64;                                          //  is not worth a gate: large n)
        ldx64 = np;
      }
      if (rc == GG_OK)
        rc = gg::trsm_packed_gated_run(n, cnt, LinvP, x64, ldx64, w.xbar, np, w.flag, 1, s);
      if (rc == GG_OK)
        rc = gg::partials_run(n, cnt, q, w.xbar, np, XLbar, np, ybar, w.P, s, w.flag, 1,
                              w.colbad);
    }
    invalid_gate = may_flag && LinvP == nullptr;   // flagged columns and no FP64 inverse
  } else {
    const double* xin = X64;
    int ldin = ldx;
    if (G8 != nullptr) {
      rc = gg::widen_run(n, cnt, G8, ldg, w.x64, np, s);
      xin = w.x64;
      ldin = np;
    }
    if (rc == GG_OK) rc = gg::trsm_packed_run(n, cnt, LinvP, xin, ldin, w.xbar, np, s);
    if (rc == GG_OK)
      rc = gg::partials_run(n, cnt, q, w.xbar, np, XLbar, np, ybar, w.P, s, nullptr, 0);
  }
  if (rc != GG_OK) return rc;
  rc = gg::reduce_solve_run(n, cnt, q, w.P, nullptr, S_TL, b_T, beta, status, sinv, s);
  if (rc == GG_OK && invalid_gate)
    rc = gg::mark_invalid_run(cnt, q + 1, w.flag, 1, beta, status, s, w.colbad);
  return rc;
}

int gg_memcpy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                      size_t height, int kind, void* stream) {
  cudaMemcpyKind k;
  switch (kind) {
    case 1: k = cudaMemcpyHostToDevice; break;
    case 2: k = cudaMemcpyDeviceToHost; break;
    case 3: k = cudaMemcpyDeviceToDevice; break;
    default:
      gg::set_error("memcpy2d: kind must be 1, 2 or 3");
      return GG_EARG;
  }
  if (height == 0 || width == 0) return GG_OK;
  GG_CUDA_TRY(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, k, as_stream(stream)));
  return GG_OK;
}

int gg_gen_genotypes_i8(unsigned long long seed, int stream_maf, int stream_geno, int n,
                        long long m, long long first, int cnt, double maf_lo, double maf_hi,
                        int8_t* G, long long ldg, double* Z, int ldz, void* stream) {
  GG_NVTX("gg_gen_genotypes_i8");
  return gg::gen_genotypes_run(seed, stream_maf, stream_geno, n, m, first, cnt, maf_lo, maf_hi, G,
                               ldg, Z, ldz, as_stream(stream));
}

}  // extern "C"
