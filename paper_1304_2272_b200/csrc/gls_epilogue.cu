// Per-SNP epilogue of the GLS sweep: reductions against the whitened covariates and the
// batched p x p SPD solve, plus the int8 -> FP64 genotype widening.
//
// Reference arithmetic (kernel.py):
//   _column_sums          kernel.py:260-270   S_BL, S_BR, b_B
//   assembly of S, rhs    kernel.py:282-289
//   cholesky_solve_batch  kernel.py:138-208   pivot rule d > p*eps*max|S| and finite,
//                                             placeholder pivot 1.0, NaN for failed systems,
//                                             optional packed S^-1 (np.tril_indices order)
// The reductions use ONE summation order for every column (lane-strided FMA chains followed by
// an xor butterfly), so a column's sums do not depend on its position in the block, and
// gram(XLbar) computed with the same kernel is bitwise consistent with S_BL/S_BR for a SNP
// column equal to a covariate column (the degenerate-SNP case, tests/conftest.py:29-41).
#include "gg_internal.cuh"

namespace gg {
namespace {

constexpr double EPS = 2.220446049250313e-16;   // 2^-52 (kernel.py:28)
constexpr int DOT_WARPS = 8;
constexpr int DOT_COLS_PER_WARP = 2;
constexpr int DOT_CHUNK = GG_TILE;   // rows of XLbar / ybar staged per step (np is a multiple)
constexpr int QMAX = GG_PMAX - 1;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

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
// Each warp owns DOT_COLS_PER_WARP columns; XLbar/ybar row chunks are staged once per CTA in
// shared memory and reused by its 8 warps.  Lane l accumulates rows l, l+32, l+64, ... in order.
template <int QM>
__device__ __forceinline__ void dots_accumulate(int np, int cnt, int q, int col0,
                                                const double* __restrict__ X, long long ldx,
                                                const double* __restrict__ XL, long long ldxl,
                                                const double* __restrict__ y, double* sm,
                                                double (&acc)[DOT_COLS_PER_WARP][QM + 2]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < DOT_COLS_PER_WARP; ++c)
#pragma unroll
    for (int k = 0; k < QM + 2; ++k) acc[c][k] = 0.0;
  for (int r0 = 0; r0 < np; r0 += DOT_CHUNK) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < (q + 1) * DOT_CHUNK; idx += blockDim.x) {
      const int k = idx / DOT_CHUNK, r = idx % DOT_CHUNK;
      sm[idx] = (k < q) ? XL[(long long)k * ldxl + r0 + r] : y[r0 + r];
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < DOT_COLS_PER_WARP; ++c) {
      const int col = col0 + c;
      if (col >= cnt) continue;
      const double* xc = X + (long long)col * ldx + r0;
#pragma unroll 4
      for (int u = 0; u < DOT_CHUNK / 32; ++u) {
        const int r = lane + 32 * u;
        const double xv = xc[r];
#pragma unroll
        for (int k = 0; k < QM; ++k)
          if (k < q) acc[c][k] = fma(xv, sm[k * DOT_CHUNK + r], acc[c][k]);
        acc[c][QM] = fma(xv, xv, acc[c][QM]);
        acc[c][QM + 1] = fma(xv, sm[q * DOT_CHUNK + r], acc[c][QM + 1]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < DOT_COLS_PER_WARP; ++c)
#pragma unroll
    for (int k = 0; k < QM + 2; ++k) acc[c][k] = warp_sum(acc[c][k]);
}

template <int QM>
__global__ void __launch_bounds__(DOT_WARPS * 32) dots_kernel(
    int np, int cnt, int q, const double* __restrict__ X, long long ldx,
    const double* __restrict__ XL, long long ldxl, const double* __restrict__ y,
    double* __restrict__ dots) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col0 = (blockIdx.x * DOT_WARPS + warp) * DOT_COLS_PER_WARP;
  double acc[DOT_COLS_PER_WARP][QM + 2];
  dots_accumulate<QM>(np, cnt, q, col0, X, ldx, XL, ldxl, y, sm, acc);
#pragma unroll
  for (int c = 0; c < DOT_COLS_PER_WARP; ++c) {
    const int col = col0 + c;
    if (col >= cnt || lane != c) continue;
    double* out = dots + (long long)col * (q + 2);
#pragma unroll
    for (int k = 0; k < QM; ++k)
      if (k < q) out[k] = acc[c][k];
    out[q] = acc[c][QM];
    out[q + 1] = acc[c][QM + 1];
  }
}

// Fused: reductions + assembly + small solve.  Lane c of each warp solves column col0 + c.
template <int QM, int PM>
__global__ void __launch_bounds__(DOT_WARPS * 32) epilogue_kernel(
    int np, int cnt, int q, const double* __restrict__ X, long long ldx,
    const double* __restrict__ XL, long long ldxl, const double* __restrict__ y,
    const double* __restrict__ S_TL, const double* __restrict__ b_T, double* __restrict__ beta,
    int* __restrict__ status, double* __restrict__ sinv) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col0 = (blockIdx.x * DOT_WARPS + warp) * DOT_COLS_PER_WARP;
  double acc[DOT_COLS_PER_WARP][QM + 2];
  dots_accumulate<QM>(np, cnt, q, col0, X, ldx, XL, ldxl, y, sm, acc);
  const int p = q + 1;
#pragma unroll
  for (int c = 0; c < DOT_COLS_PER_WARP; ++c) {
    const int col = col0 + c;
    if (col >= cnt || lane != c) continue;
    double S[PM * PM], rhs[PM], x[PM];
    for (int i = 0; i < q; ++i)
      for (int j = 0; j < q; ++j) S[i * PM + j] = S_TL[i * q + j];
#pragma unroll
    for (int k = 0; k < QM; ++k)
      if (k < q) {
        S[q * PM + k] = acc[c][k];
        S[k * PM + q] = acc[c][k];
        rhs[k] = b_T[k];
      }
    S[q * PM + q] = acc[c][QM];
    rhs[q] = acc[c][QM + 1];
    double* so = sinv ? sinv + (long long)col * (p * (p + 1) / 2) : nullptr;
    status[col] = small_spd_solve<PM>(p, S, rhs, x, so);
    for (int i = 0; i < p; ++i) beta[(long long)col * p + i] = x[i];
  }
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

size_t dot_smem(int q) { return (size_t)(q + 1) * DOT_CHUNK * sizeof(double); }
int dot_grid(int cnt) {
  return (cnt + DOT_WARPS * DOT_COLS_PER_WARP - 1) / (DOT_WARPS * DOT_COLS_PER_WARP);
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

int dots_run(int n, int cnt, int q, const double* Xbar, int ldx, const double* XLbar, int ldxl,
             const double* ybar, double* dots, cudaStream_t s) {
  if (q < 0 || q > QMAX || n < 1) {
    set_error("dots: need 0 <= q <= 19 and n >= 1");
    return GG_EARG;
  }
  if (cnt <= 0) return GG_OK;
  int rc = check_ld(n, ldx, q > 0 ? ldxl : pad_rows(n));
  if (rc != GG_OK) return rc;
  const int np = pad_rows(n);
  const size_t sm = dot_smem(q);
  if (q <= 3) {
    dots_kernel<3><<<dot_grid(cnt), DOT_WARPS * 32, sm, s>>>(np, cnt, q, Xbar, ldx, XLbar, ldxl,
                                                            ybar, dots);
  } else if (q <= 7) {
    dots_kernel<7><<<dot_grid(cnt), DOT_WARPS * 32, sm, s>>>(np, cnt, q, Xbar, ldx, XLbar, ldxl,
                                                            ybar, dots);
  } else {
    GG_CUDA_TRY(cudaFuncSetAttribute(dots_kernel<QMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sm));
    dots_kernel<QMAX><<<dot_grid(cnt), DOT_WARPS * 32, sm, s>>>(np, cnt, q, Xbar, ldx, XLbar,
                                                               ldxl, ybar, dots);
  }
  GG_LAUNCH_CHECK("dots_kernel");
  return GG_OK;
}

int epilogue_run(int n, int cnt, int q, const double* Xbar, int ldx, const double* XLbar,
                 int ldxl, const double* ybar, const double* S_TL, const double* b_T,
                 double* beta, int* status, double* sinv, cudaStream_t s) {
  if (q < 0 || q > QMAX || n < 1) {
    set_error("epilogue: need 0 <= q <= 19 and n >= 1");
    return GG_EARG;
  }
  if (cnt <= 0) return GG_OK;
  int rc = check_ld(n, ldx, q > 0 ? ldxl : pad_rows(n));
  if (rc != GG_OK) return rc;
  const int np = pad_rows(n);
  const size_t sm = dot_smem(q);
  const int grid = dot_grid(cnt);
  if (q <= 3) {
    epilogue_kernel<3, 4><<<grid, DOT_WARPS * 32, sm, s>>>(np, cnt, q, Xbar, ldx, XLbar, ldxl, ybar,
                                                           S_TL, b_T, beta, status, sinv);
  } else if (q <= 7) {
    epilogue_kernel<7, 8><<<grid, DOT_WARPS * 32, sm, s>>>(np, cnt, q, Xbar, ldx, XLbar, ldxl, ybar,
                                                           S_TL, b_T, beta, status, sinv);
  } else {
    GG_CUDA_TRY(cudaFuncSetAttribute(epilogue_kernel<QMAX, GG_PMAX>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    epilogue_kernel<QMAX, GG_PMAX><<<grid, DOT_WARPS * 32, sm, s>>>(
        np, cnt, q, Xbar, ldx, XLbar, ldxl, ybar, S_TL, b_T, beta, status, sinv);
  }
  GG_LAUNCH_CHECK("epilogue_kernel");
  return GG_OK;
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
