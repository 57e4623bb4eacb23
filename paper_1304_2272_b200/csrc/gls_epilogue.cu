// Per-SNP epilogue of the GLS sweep: reductions against the whitened covariates and the
// batched p x p SPD solve, plus the int8 -> FP64 genotype widening.
//
// Reference arithmetic (kernel.py):
//   _column_sums          kernel.py:260-270   S_BL, S_BR, b_B
//   assembly of S, rhs    kernel.py:282-289
//   cholesky_solve_batch  kernel.py:138-208   pivot rule d > p*eps*max|S| and finite,
//                                             placeholder pivot 1.0, NaN for failed systems,
//                                             optional packed S^-1 (np.tril_indices order)
// Canonical reduction order (shared with the fused epilogue of the int8 TRSM, trsm_i8.cu):
//   partial_rb = FMA chain over the 32 rows of row block rb, in order;
//   lane_l     = sum of partial_rb for rb = l, l+32, l+64, ... in order (l = 0..31);
//   dot        = xor-butterfly sum of the 32 lane values (identical on every lane).
// Every column uses this order whatever its position, and gram(XLbar) / S_TL / b_T are formed
// the same way, so a SNP column equal to a covariate column yields an exactly singular S (the
// degenerate-SNP case, tests/conftest.py:29-41).  Two kernels: partials (per column and row
// block; or written directly by the int8 TRSM epilogue) and reduce+solve (per column).
#include "gg_internal.cuh"

namespace gg {
namespace {

constexpr double EPS = 2.220446049250313e-16;   // 2^-52 (kernel.py:28)
constexpr int QMAX = GG_PMAX - 1;
constexpr int RB = GG_DOT_BLOCK;   // rows per partial (np is a multiple)

// ---- small SPD solve, mirroring cholesky_solve_batch operation by operation -------------
// S, L: p x p row-major local arrays (stride PM).  Products and differences are rounded
// separately (__dmul_rn/__dsub_rn), as in the reference's numpy expressions.
template <int PM>
__device__ void small_factor(int p, const double* S, double* L, bool& ok, int& first_bad) {
  double mx = 0.0;
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) mx = fmax(mx, fabs(S[i * PM + j]));
  const double thresh = __dmul_rn(__dmul_rn((double)p, EPS), mx);
  ok = true;
  first_bad = -1;
  for (int j = 0; j < p; ++j) {
    double d = S[j * PM + j];
    if (j > 0) {
      double t = __dmul_rn(L[j * PM + 0], L[j * PM + 0]);
      for (int k = 1; k < j; ++k) t = __dadd_rn(t, __dmul_rn(L[j * PM + k], L[j * PM + k]));
      d = __dsub_rn(d, t);
    }
    const bool good = isfinite(d) && d > thresh;
    if (!good && ok) first_bad = j;
    ok = ok && good;
    if (!good) d = 1.0;   // placeholder pivot keeps the math finite (kernel.py:160)
    const double ljj = sqrt(d);
    L[j * PM + j] = ljj;
    for (int i = j + 1; i < p; ++i) {
      double s = S[i * PM + j];
      if (j > 0) {
        double t = __dmul_rn(L[i * PM + 0], L[j * PM + 0]);
        for (int k = 1; k < j; ++k) t = __dadd_rn(t, __dmul_rn(L[i * PM + k], L[j * PM + k]));
        s = __dsub_rn(s, t);
      }
      L[i * PM + j] = __ddiv_rn(s, ljj);
    }
  }
}

template <int PM>
__device__ void small_solve_factored(int p, const double* L, const double* b, double* x) {
  double z[PM];
  for (int i = 0; i < p; ++i) {
    double acc = b[i];
    for (int k = 0; k < i; ++k) acc = __dsub_rn(acc, __dmul_rn(L[i * PM + k], z[k]));
    z[i] = __ddiv_rn(acc, L[i * PM + i]);
  }
  for (int i = p - 1; i >= 0; --i) {
    double acc = z[i];
    for (int k = i + 1; k < p; ++k) acc = __dsub_rn(acc, __dmul_rn(L[k * PM + i], x[k]));
    x[i] = __ddiv_rn(acc, L[i * PM + i]);
  }
}

// Solve one system; writes x (p), optional packed inverse; returns first failing pivot or -1.
template <int PM>
__device__ int small_spd_solve(int p, const double* S, const double* rhs, double* x_out,
                               double* sinv_out) {
  double L[PM * PM];
  bool ok;
  int bad;
  small_factor<PM>(p, S, L, ok, bad);
  double x[PM];
  small_solve_factored<PM>(p, L, rhs, x);
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  for (int i = 0; i < p; ++i) x_out[i] = ok ? x[i] : qnan;
  if (sinv_out != nullptr) {
    // column c of S^-1 from e_c; packed lower triangle in np.tril_indices order
    double inv[PM * PM];
    for (int c = 0; c < p; ++c) {
      double e[PM], col[PM];
      for (int i = 0; i < p; ++i) e[i] = (i == c) ? 1.0 : 0.0;
      small_solve_factored<PM>(p, L, e, col);
      for (int i = 0; i < p; ++i) inv[i * PM + c] = col[i];
    }
    int idx = 0;
    for (int i = 0; i < p; ++i)
      for (int j = 0; j <= i; ++j) sinv_out[idx++] = ok ? inv[i * PM + j] : qnan;
  }
  return ok ? -1 : bad;
}

// ---- reductions ----------------------------------------------------------------------------
// partials[(rb * (q+2) + k) * cnt + col]: k < q -> x.XL[:,k], q -> x.x, q+1 -> x.y over the
// 32-row block rb (layout shared with the fused epilogue of trsm_i8.cu).
// CTA = 8 warps = 8 columns x 32 row blocks (1024 rows): XL/y rows staged once per CTA, each
// warp stages its column's 1024 values (coalesced, padded against bank conflicts) and lane l
// computes row block l's partial with one sequential FMA chain per output.
constexpr int PRB = 32;               // row blocks per CTA (one per lane)
constexpr int PROWS = PRB * RB;       // 1024 rows
template <int QM, int PCOLS>          // PCOLS columns per CTA (one per warp)
__global__ void __launch_bounds__(PCOLS * 32) partials_kernel(
    int nrb, int cnt, int q, const double* __restrict__ X, long long ldx,
    const double* __restrict__ XL, long long ldxl, const double* __restrict__ y,
    double* __restrict__ P, const int* gate, int gate_value, const int* __restrict__ colmask) {
  if (gate != nullptr && *gate != gate_value) return;
  extern __shared__ double sm[];
  constexpr int LDP = PROWS + PRB;                   // padded: row r at r + r / RB
  double* sv = sm;                                   // (q+1) x LDP: XL columns, then y
  double* sx = sm + (size_t)(q + 1) * LDP;           // PCOLS x LDP: the warps' columns
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb0 = blockIdx.y * PRB;
  const long long r0 = (long long)rb0 * RB;
  const int nrows = min(PROWS, (nrb - rb0) * RB);
  for (int idx = threadIdx.x; idx < (q + 1) * nrows; idx += blockDim.x) {
    const int k = idx / nrows, r = idx % nrows;
    sv[k * LDP + r + r / RB] = (k < q) ? XL[k * ldxl + r0 + r] : y[r0 + r];
  }
  const int col = blockIdx.x * PCOLS + warp;
  double* mx = sx + warp * LDP;
  if (col < cnt) {
    const double* xc = X + (long long)col * ldx + r0;
    for (int r = lane; r < nrows; r += 32) mx[r + r / RB] = xc[r];
  }
  __syncthreads();
  const int rb = rb0 + lane;
  if (col >= cnt || rb >= nrb) return;
  if (colmask != nullptr && colmask[col] == 0) return;   // column computed by another path
  const double* xr = mx + lane * (RB + 1);
  double acc[QM + 2];
#pragma unroll
  for (int k = 0; k < QM + 2; ++k) acc[k] = 0.0;
  for (int i = 0; i < RB; ++i) {
    const double xv = xr[i];
    const int r = lane * (RB + 1) + i;
#pragma unroll
    for (int k = 0; k < QM; ++k)
      if (k < q) acc[k] = fma(xv, sv[k * LDP + r], acc[k]);
    acc[QM] = fma(xv, xv, acc[QM]);
    acc[QM + 1] = fma(xv, sv[q * LDP + r], acc[QM + 1]);
  }
  double* out = P + (long long)rb * (q + 2) * cnt + col;   // value-major: coalesced over col
#pragma unroll
  for (int k = 0; k < QM; ++k)
    if (k < q) out[(long long)k * cnt] = acc[k];
  out[(long long)q * cnt] = acc[QM];
  out[(long long)(q + 1) * cnt] = acc[QM + 1];
}

// Cross-block part of the canonical order: "lane" l sums the partials of row blocks l, l+32,
// l+64, ... in order, then an xor butterfly combines the 32 lane sums (the value a warp reduction
// v += shfl_xor(v, o), o = 16 .. 1, leaves on every lane); then (if S_TL is given) the SNP's
// S = [[S_TL, S_BL^T], [S_BL, S_BR]], rhs = [b_T, b_B] is assembled and solved.

// 32 columns per CTA.  Warp w sums, for every column at once (coalesced loads of consecutive
// columns' partials), the row blocks of lane slots l = w, w+8, w+16, w+24 -- exactly lane l's
// share of the canonical order -- into shared memory; warp 0 then applies the xor-butterfly tree
// (t_l <- t_l + t_(l^o), o = 16 .. 1) per column and value, and solves.
#ifndef RS_WARPS_N
#define RS_WARPS_N 8
#endif
#ifndef RS_UNROLL
#define RS_UNROLL 6
#endif
#ifndef RS_MINB
#define RS_MINB 2
#endif
#define RS_PRAGMA_(x) _Pragma(#x)
#define RS_PRAGMA_UNROLL(n) RS_PRAGMA_(unroll n)
constexpr int RS_WARPS = RS_WARPS_N;   // warps per 32-SNP block: each takes the lane slots l = warp, warp + 8, ..
                               // (r02 end: RS_UNROLL row blocks of loads in flight per slot -- the kernel is
                               // HBM-latency-bound; two blocks per SM so that all 256 blocks of an
                               // 8,192-SNP launch are resident at once; same sums in the same order)
template <int QM, int PM>
__global__ void __launch_bounds__(RS_WARPS * 32, RS_MINB) reduce_solve_kernel(
    int nrb, int cnt, int q, const double* __restrict__ P, double* __restrict__ dots,
    const double* __restrict__ S_TL, const double* __restrict__ b_T, double* __restrict__ beta,
    int* __restrict__ status, double* __restrict__ sinv) {
  extern __shared__ double sh[];   // [32 lane slots][32 columns][QM + 2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = blockIdx.x * 32 + lane;
  const long long stride = (long long)cnt * (q + 2);
  for (int l = warp; l < 32; l += RS_WARPS) {
    double acc[QM + 2];
#pragma unroll
    for (int k = 0; k < QM + 2; ++k) acc[k] = 0.0;
    if (col < cnt) {
      RS_PRAGMA_UNROLL(RS_UNROLL)
      for (int rb = l; rb < nrb; rb += 32) {
        const double* pp = P + rb * stride + col;           // value-major, coalesced over col
#pragma unroll
        for (int k = 0; k < QM; ++k)
          if (k < q) acc[k] = acc[k] + pp[(long long)k * cnt];
        acc[QM] = acc[QM] + pp[(long long)q * cnt];
        acc[QM + 1] = acc[QM + 1] + pp[(long long)(q + 1) * cnt];
      }
    }
    double* dst = sh + (l * 32 + lane) * (QM + 2);
#pragma unroll
    for (int k = 0; k < QM + 2; ++k) dst[k] = acc[k];
  }
  __syncthreads();
  if (warp != 0 || col >= cnt) return;
  double tot[QM + 2];
#pragma unroll 1
  for (int k = 0; k < QM + 2; ++k) {
    double t[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) t[l] = sh[(l * 32 + lane) * (QM + 2) + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double u[32];
#pragma unroll
      for (int l = 0; l < 32; ++l) u[l] = t[l] + t[l ^ o];
#pragma unroll
      for (int l = 0; l < 32; ++l) t[l] = u[l];
    }
    tot[k] = t[0];
  }
  if (dots != nullptr) {
    double* out = dots + (long long)col * (q + 2);
#pragma unroll
    for (int k = 0; k < QM; ++k)
      if (k < q) out[k] = tot[k];
    out[q] = tot[QM];
    out[q + 1] = tot[QM + 1];
  }
  if (beta == nullptr) return;
  const int p = q + 1;
  double S[PM * PM], rhs[PM], x[PM];
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) S[i * PM + j] = S_TL[i * q + j];
#pragma unroll
  for (int k = 0; k < QM; ++k)
    if (k < q) {
      S[q * PM + k] = tot[k];
      S[k * PM + q] = tot[k];
      rhs[k] = b_T[k];
    }
  S[q * PM + q] = tot[QM];
  rhs[q] = tot[QM + 1];
  double* so = sinv ? sinv + (long long)col * (p * (p + 1) / 2) : nullptr;
  status[col] = small_spd_solve<PM>(p, S, rhs, x, so);
  for (int i = 0; i < p; ++i) beta[(long long)col * p + i] = x[i];
}

template <int PM>
__global__ void small_solve_kernel(int batch, int p, const double* __restrict__ S,
                                   const double* __restrict__ rhs, double* __restrict__ x,
                                   int* __restrict__ status, double* __restrict__ sinv) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double Sl[PM * PM], r[PM], xo[PM];
  for (int i = 0; i < p; ++i) {
    for (int j = 0; j < p; ++j) Sl[i * PM + j] = S[(long long)b * p * p + i * p + j];
    r[i] = rhs[(long long)b * p + i];
  }
  double* so = sinv ? sinv + (long long)b * (p * (p + 1) / 2) : nullptr;
  status[b] = small_spd_solve<PM>(p, Sl, r, xo, so);
  for (int i = 0; i < p; ++i) x[(long long)b * p + i] = xo[i];
}

// Rejection (device-side): if *gate == gate_value every SNP of the block (or, with colmask, every
// flagged SNP) gets status GG_STATUS_INVALID and NaN coefficients (values the selected path cannot compute exactly
// and no FP64 inverse to fall back on).
__global__ void mark_invalid_kernel(int cnt, int p, const int* __restrict__ gate, int gate_value,
                                    double* __restrict__ beta, int* __restrict__ status,
                                    const int* __restrict__ colmask) {
  if (*gate != gate_value) return;
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)cnt * p;
       e += (long long)gridDim.x * blockDim.x) {
    if (colmask != nullptr && colmask[e / p] == 0) continue;   // only the flagged columns
    beta[e] = qnan;
    if (e % p == 0) status[e / p] = GG_STATUS_INVALID;
  }
}

__global__ void widen_kernel(int n, int np, int cnt, const int8_t* __restrict__ G, long long ldg,
                             double* __restrict__ X, long long ldx) {
  const long long total = (long long)np * cnt;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % np);
    const long long j = idx / np;
    X[i + j * ldx] = (i < n) ? (double)G[i + j * ldg] : 0.0;
  }
}

int check_ld(int n, int ldx, int ldxl) {
  const int np = pad_rows(n);
  if (ldx < np || ldxl < np) {
    set_error("leading dimension must be >= gg_pad(n)");
    return GG_EDIM;
  }
  return GG_OK;
}

}  // namespace

template <int QM, int PC>
static int launch_partials(int nrb, int cnt, int q, const double* Xbar, int ldx,
                           const double* XLbar, int ldxl, const double* ybar, double* P,
                           cudaStream_t s, const int* gate, int gate_value,
                           const int* colmask) {
  dim3 grid((cnt + PC - 1) / PC, (nrb + PRB - 1) / PRB);
  const size_t sm = (size_t)(q + 1 + PC) * (PROWS + PRB) * sizeof(double);
  GG_CUDA_TRY(cudaFuncSetAttribute(partials_kernel<QM, PC>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  partials_kernel<QM, PC><<<grid, PC * 32, sm, s>>>(nrb, cnt, q, Xbar, ldx, XLbar, ldxl, ybar, P,
                                                    gate, gate_value, colmask);
  GG_LAUNCH_CHECK("partials_kernel");
  return GG_OK;
}

int partials_run(int n, int cnt, int q, const double* Xbar, int ldx, const double* XLbar,
                 int ldxl, const double* ybar, double* P, cudaStream_t s, const int* gate,
                 int gate_value, const int* colmask) {
  const int nrb = pad_rows(n) / RB;
  if (q <= 3)
    return launch_partials<3, 8>(nrb, cnt, q, Xbar, ldx, XLbar, ldxl, ybar, P, s, gate,
                                 gate_value, colmask);
  if (q <= 7)
    return launch_partials<7, 8>(nrb, cnt, q, Xbar, ldx, XLbar, ldxl, ybar, P, s, gate,
                                 gate_value, colmask);
  return launch_partials<QMAX, 4>(nrb, cnt, q, Xbar, ldx, XLbar, ldxl, ybar, P, s, gate,
                                  gate_value, colmask);
}

template <int QM, int PM>
static int launch_reduce(int nrb, int cnt, int q, const double* P, double* dots,
                         const double* S_TL, const double* b_T, double* beta, int* status,
                         double* sinv, cudaStream_t s) {
  const size_t sm = (size_t)32 * 32 * (QM + 2) * sizeof(double);
  GG_CUDA_TRY(cudaFuncSetAttribute(reduce_solve_kernel<QM, PM>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  reduce_solve_kernel<QM, PM><<<(cnt + 31) / 32, RS_WARPS * 32, sm, s>>>(nrb, cnt, q, P, dots, S_TL, b_T,
                                                                beta, status, sinv);
  GG_LAUNCH_CHECK("reduce_solve_kernel");
  return GG_OK;
}

int mark_invalid_run(int cnt, int p, const int* gate, int gate_value, double* beta, int* status,
                     cudaStream_t s, const int* colmask) {
  if (cnt <= 0) return GG_OK;
  const int grid = (int)(((long long)cnt * p + 255) / 256 > 1184 ? 1184 : ((long long)cnt * p + 255) / 256);
  mark_invalid_kernel<<<grid, 256, 0, s>>>(cnt, p, gate, gate_value, beta, status, colmask);
  GG_LAUNCH_CHECK("mark_invalid_kernel");
  return GG_OK;
}

int reduce_solve_run(int n, int cnt, int q, const double* P, double* dots, const double* S_TL,
                     const double* b_T, double* beta, int* status, double* sinv, cudaStream_t s) {
  const int nrb = pad_rows(n) / RB;
  if (q <= 3) return launch_reduce<3, 4>(nrb, cnt, q, P, dots, S_TL, b_T, beta, status, sinv, s);
  if (q <= 7) return launch_reduce<7, 8>(nrb, cnt, q, P, dots, S_TL, b_T, beta, status, sinv, s);
  return launch_reduce<QMAX, GG_PMAX>(nrb, cnt, q, P, dots, S_TL, b_T, beta, status, sinv, s);
}

size_t partials_bytes(int n, int cnt, int q) {
  return (size_t)(pad_rows(n) / RB) * (size_t)cnt * (size_t)(q + 2) * sizeof(double);
}

int dots_run(int n, int cnt, int q, const double* Xbar, int ldx, const double* XLbar, int ldxl,
             const double* ybar, double* dots, double* P, cudaStream_t s) {
  if (q < 0 || q > QMAX || n < 1) {
    set_error("dots: need 0 <= q <= 19 and n >= 1");
    return GG_EARG;
  }
  if (cnt <= 0) return GG_OK;
  int rc = check_ld(n, ldx, q > 0 ? ldxl : pad_rows(n));
  if (rc != GG_OK) return rc;
  rc = partials_run(n, cnt, q, Xbar, ldx, XLbar, ldxl, ybar, P, s, nullptr, 0);
  if (rc == GG_OK)
    rc = reduce_solve_run(n, cnt, q, P, dots, nullptr, nullptr, nullptr, nullptr, nullptr, s);
  return rc;
}

int epilogue_run(int n, int cnt, int q, const double* Xbar, int ldx, const double* XLbar,
                 int ldxl, const double* ybar, const double* S_TL, const double* b_T,
                 double* beta, int* status, double* sinv, double* P, cudaStream_t s) {
  if (q < 0 || q > QMAX || n < 1) {
    set_error("epilogue: need 0 <= q <= 19 and n >= 1");
    return GG_EARG;
  }
  if (cnt <= 0) return GG_OK;
  int rc = check_ld(n, ldx, q > 0 ? ldxl : pad_rows(n));
  if (rc != GG_OK) return rc;
  rc = partials_run(n, cnt, q, Xbar, ldx, XLbar, ldxl, ybar, P, s, nullptr, 0);
  if (rc == GG_OK)
    rc = reduce_solve_run(n, cnt, q, P, nullptr, S_TL, b_T, beta, status, sinv, s);
  return rc;
}

int small_solve_run(int batch, int p, const double* S, const double* rhs, double* x, int* status,
                    double* sinv, cudaStream_t s) {
  if (p < 1 || p > GG_PMAX) {
    set_error("small_spd_solve: need 1 <= p <= 20");
    return GG_EARG;
  }
  if (batch <= 0) return GG_OK;
  const int threads = 128, grid = (batch + threads - 1) / threads;
  if (p <= 4) small_solve_kernel<4><<<grid, threads, 0, s>>>(batch, p, S, rhs, x, status, sinv);
  else if (p <= 8) small_solve_kernel<8><<<grid, threads, 0, s>>>(batch, p, S, rhs, x, status, sinv);
  else small_solve_kernel<GG_PMAX><<<grid, threads, 0, s>>>(batch, p, S, rhs, x, status, sinv);
  GG_LAUNCH_CHECK("small_solve_kernel");
  return GG_OK;
}

int widen_run(int n, int cnt, const int8_t* G, long long ldg, double* X, int ldx, cudaStream_t s) {
  const int np = pad_rows(n);
  if (ldg < n || ldx < np) {
    set_error("widen: ldg >= n and ldx >= gg_pad(n) required");
    return GG_EDIM;
  }
  if (cnt <= 0) return GG_OK;
  long long total = (long long)np * cnt;
  long long grid = (total + 255) / 256;
  if (grid > 148 * 32) grid = 148 * 32;
  widen_kernel<<<(int)grid, 256, 0, s>>>(n, np, cnt, G, ldg, X, ldx);
  GG_LAUNCH_CHECK("widen_kernel");
  return GG_OK;
}

}  // namespace gg
