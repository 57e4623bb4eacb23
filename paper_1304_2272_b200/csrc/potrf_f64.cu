// Blocked FP64 Cholesky (right-looking, nb = 128) fused with the triangular inverse.
//
// Replaces kernel.cholesky_spd (reference kernel.py:92-109: LAPACK dpotrf lower, clean=1).
// Per 128-column block k:
//   leaf     : one CTA factors the 128x128 diagonal block in shared memory, blocked by 32
//              (pivot rule of LAPACK dpotf2: fail iff a_jj <= 0 or NaN) and inverts it
//              (Dinv_k = L_kk^-1, written to the diagonal block of Linv);
//   panel    : L21 = A21 * Dinv_k^T                 (DMMA GEMM, op(B) = B^T)
//   trailing : A22 -= L21 * L21^T, lower tiles only  (DMMA GEMM, K = 128)
// then the off-diagonal blocks of Linv by the recursive formula
//   inv([A 0; B C]) = [A^-1 0; -C^-1 B A^-1  C^-1]
// with triangular-aware DMMA GEMMs.  A failing pivot sets a device flag that turns every later
// kernel into a no-op; the host reads it once at the end (no per-block synchronisation).
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "gg_internal.cuh"

namespace gg {
namespace {

constexpr int NB = 128;
constexpr int OUTER = 8 * NB;   // outer block width of the two-level Cholesky
constexpr bool OZAKI_DEFAULT = true;
constexpr int LEAF_THREADS = 384;

struct PotrfHeader {
  int info;                      // 0 = ok, else failing pivot + 1
  int pad_;
  unsigned long long nonfinite;  // min row-major index of a non-finite entry
};
constexpr size_t HDR_BYTES = 256;

// The factor's input pass: L = lower(M) extended by the identity on the padding block, Linv
// zeroed, and the first non-finite entry of M in row-major order (kernel.py:101-103 reports its
// row) -- one pass over M through 32 x 32 shared-memory tiles: M is read along its contiguous
// dimension (row-major input: a C-contiguous array) and L written column-major, both coalesced
// (element-wise forms re-read a row-major M ~9x from DRAM: 119 GB at n = 4e4).
__global__ void __launch_bounds__(256) init_factor_tiled_kernel(
    int n, int np, const double* __restrict__ M, long long rs, long long cs,
    double* __restrict__ L, double* __restrict__ Linv, long long ldp,
    unsigned long long* first) {
  __shared__ double t[32][33];
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const bool rowmaj = cs == 1;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  unsigned long long bad = ~0ull;
  for (int k = ty; k < 32; k += 8) {
    const int i = rowmaj ? i0 + k : i0 + tx, j = rowmaj ? j0 + tx : j0 + k;
    double v = 0.0;
    if (i < n && j < n) {
      v = M[i * rs + j * cs];
      if (!isfinite(v)) bad = min(bad, (unsigned long long)i * n + j);
    }
    if (rowmaj)
      t[k][tx] = v;
    else
      t[tx][k] = v;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int i = i0 + tx, j = j0 + k;
    double v;
    if (i < n && j < n) v = (i >= j) ? t[tx][k] : 0.0;
    else v = (i == j) ? 1.0 : 0.0;   // identity extension on the padding block
    L[i + (long long)j * ldp] = v;
    if (Linv != nullptr) Linv[i + (long long)j * ldp] = 0.0;
  }
  if (bad != ~0ull) atomicMin(first, bad);
}

__global__ void zero_square_kernel(int np, double* __restrict__ A, long long ld) {
  const long long total = (long long)np * np;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % np), j = (int)(idx / np);
    A[i + j * ld] = 0.0;
  }
}

// ---- 128 x 128 leaf: factor + inverse of one diagonal block, one CTA (12 warps) ----------------
// S = the block in shared memory, row-major with row stride LDS = 132 doubles (= 4 mod 16: the
// DMMA fragment reads S[r0+g][k+t] and S[k+t][c0+g] of a warp are bank-conflict free).
// Factor, per 32-column sub-block J (right-looking):
//   * warp 0 factors S_JJ in registers (lane = row; LAPACK dpotf2's pivot rule: fail iff the
//     pivot is <= 0 or NaN), writes L_JJ to global memory and overwrites S_JJ with
//     T_J = L_JJ^-1 (lane = column, column-oriented substitution: one FMA per step on the
//     dependent chain, not a dot product);
//   * panel L_IJ = S_IJ T_J^T and trailing update S_II' -= L_IJ L_I'J^T on the FP64 tensor
//     cores (mma.sync m8n8k4 -> DMMA), one 8 x 8 output tile per warp at a time.
// S then holds [T_0; L_10 T_1; L_20 L_21 T_2; L_30 L_31 L_32 T_3].  Inverse X = L^-1 by the
// recursion inv([A 0; B C]) = [A^-1 0; -C^-1 B A^-1  C^-1] on 32- then 64-blocks, in place:
//   X_10 = -T_1 (L_10 T_0), X_32 = -T_3 (L_32 T_2);   X[64:, :64] = -X_C (L[64:, :64] X_A)
// -- four DMMA phases.  (r01/r02 leaf: DFMA loops and dot-product substitutions, 148 us per
// launch, 31k SASS instructions; this one keeps the dependent chains to the 128 pivots.)
constexpr int LB = 32;                  // sub-block edge
constexpr int LDS = NB + 4;             // S row stride (doubles)
constexpr int WLD = 64 + 4;             // scratch W row stride
constexpr int LEAF_WARPS = LEAF_THREADS / 32;
constexpr size_t LEAF_SMEM = (size_t)(NB * LDS + 64 * WLD) * sizeof(double) + 16;
constexpr unsigned FULL = 0xffffffffu;

// D(8x8) += A(8x4) B(4x8); lane (g = lane>>2, t = lane&3) holds A[g][t], B[t][g], D[g][2t..2t+1]
__device__ __forceinline__ void dmma_leaf(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// acc = sum_{k in [kb, ke)} X[r0+g][k] Y(k, c0+g): Y(k, c) = Y[c][k] (YT) or Y[k][c]; kb, ke % 4 == 0
template <bool YT>
__device__ __forceinline__ void tile8(double (&acc)[2], const double* X, int ldx, int r0,
                                      const double* Y, int ldy, int c0, int kb, int ke, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const double* xp = X + (r0 + g) * ldx + t;
  const double* yp = YT ? Y + (c0 + g) * ldy + t : Y + t * ldy + c0 + g;
  acc[0] = acc[1] = 0.0;
#pragma unroll 4
  for (int k = kb; k < ke; k += 4) dmma_leaf(acc, xp[k], YT ? yp[k] : yp[k * ldy]);
}

// warp: factor the 32 x 32 lower block held row-per-lane in r (right-looking); returns the
// failing local column or -1.  The scaling uses 1/sqrt(d) (dpotf2 scales by the reciprocal pivot).
__device__ __forceinline__ int warp_factor32(double (&r)[LB], int lane) {
  int fail = -1;
#pragma unroll
  for (int j = 0; j < LB; ++j) {
    double d = __shfl_sync(FULL, r[j], j);
    if (fail < 0 && !(d > 0.0)) fail = j;        // uniform: every lane sees the same d
    if (fail >= 0) d = 1.0;                      // keep the arithmetic finite past a failure
    // the scale must be the rounded reciprocal of the stored pivot (dpotf2): rsqrt(d) instead
    // measured 10x larger GLS errors on AR(1) covariances (rho = 0.999: 5.3e-10 vs 5.1e-11)
    const double piv = sqrt(d), rs = 1.0 / piv;
    if (lane == j) r[j] = piv;
    else if (lane > j) r[j] *= rs;
#pragma unroll
    for (int c = 0; c < LB; ++c) {   // constant bounds: fully unrolled, r[] stays in registers
      if (c > j) {
        const double lc = __shfl_sync(FULL, r[j], c);
        if (lane >= c) r[c] -= r[j] * lc;
      }
    }
  }
  return fail;
}

// warp: column `lane` of T = L^-1 for the 32 x 32 lower block at S + j0 (j0 + j0 LDS), by
// column-oriented substitution (L read by broadcast); t[i] = T[i][lane]
__device__ __forceinline__ void warp_inverse32(const double* S, int j0, double (&t)[LB], int lane) {
  const double* Lb = S + j0 * LDS + j0;
  const double rdl = 1.0 / Lb[lane * LDS + lane];
#pragma unroll
  for (int i = 0; i < LB; ++i) t[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < LB; ++k) {
    t[k] *= __shfl_sync(FULL, rdl, k);
#pragma unroll
    for (int i = 0; i < LB; ++i)
      if (i > k) t[i] -= Lb[i * LDS + k] * t[k];
  }
}

template <bool FACTOR>
__global__ void __launch_bounds__(LEAF_THREADS, 1) leaf_kernel(double* A, long long ld,
                                                               double* Dinv, long long ldi, int k0,
                                                               int* info, int panel = 0) {
  extern __shared__ double lsm[];
  double* S = lsm;                          // 128 x LDS
  double* W = lsm + NB * LDS;               // 64 x WLD scratch
  int* fail = reinterpret_cast<int*>(W + 64 * WLD);
  if (info != nullptr && *info != 0) return;
  if (!FACTOR) k0 = blockIdx.x * NB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  double* Ab = A + k0 + (long long)k0 * ld;
  for (int e = tid; e < NB * NB; e += LEAF_THREADS) {   // column-major global -> row-major smem
    const int r = e % NB, c = e / NB;
    S[r * LDS + c] = (r >= c) ? Ab[r + (long long)c * ld] : 0.0;
  }
  if (tid == 0) *fail = -1;
  __syncthreads();
  if (FACTOR) {
    for (int J = 0; J < NB / LB; ++J) {
      const int j0 = J * LB;
      if (warp == 0) {
        double r[LB];
#pragma unroll
        for (int c = 0; c < LB; ++c) r[c] = S[(j0 + lane) * LDS + j0 + c];
        const int f = warp_factor32(r, lane);
        if (f >= 0) {
          if (lane == 0) *fail = j0 + f;
        } else {
#pragma unroll
          for (int c = 0; c < LB; ++c) {
            S[(j0 + lane) * LDS + j0 + c] = r[c];
            Ab[(j0 + lane) + (long long)(j0 + c) * ld] = (lane >= c) ? r[c] : 0.0;
          }
          __syncwarp();
          double tc[LB];
          warp_inverse32(S, j0, tc, lane);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < LB; ++i) S[(j0 + i) * LDS + j0 + lane] = tc[i];
        }
      }
      __syncthreads();
      if (*fail >= 0) {
        if (tid == 0) *info = k0 + *fail + 1;
        return;
      }
      const int m = (NB - j0 - LB) / 8;     // 8-row tiles below the diagonal block
      if (m == 0) break;
      // panel L_IJ = S_IJ T_J^T: warp w owns row tile w (all its 32 columns; in place)
      if (warp < m) {
        const int r0 = j0 + LB + 8 * warp;
        double a[LB / 4], out[4][2];
#pragma unroll
        for (int kk = 0; kk < LB / 4; ++kk) a[kk] = S[(r0 + g) * LDS + j0 + 4 * kk + t4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          out[nt][0] = out[nt][1] = 0.0;
#pragma unroll
          for (int kk = 0; kk <= 2 * nt + 1; ++kk)   // T_J[c][k] = 0 for k > c
            dmma_leaf(out[nt], a[kk], S[(j0 + 8 * nt + g) * LDS + j0 + 4 * kk + t4]);
        }
        __syncwarp();
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) S[(r0 + g) * LDS + j0 + 8 * nt + 2 * t4 + e] = out[nt][e];
      }
      __syncthreads();
      // trailing update of the lower part: S_II' -= L_IJ L_I'J^T (lower 8 x 8 tiles)
      for (int tt = warp; tt < m * (m + 1) / 2; tt += LEAF_WARPS) {
        int rt = 0;
        while ((rt + 1) * (rt + 2) / 2 <= tt) ++rt;
        const int ct = tt - rt * (rt + 1) / 2;
        const int r0 = j0 + LB + 8 * rt, c0 = j0 + LB + 8 * ct;
        double acc[2];
        tile8<true>(acc, S + j0, LDS, r0, S + j0, LDS, c0, 0, LB, lane);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int row = r0 + g, col = c0 + 2 * t4 + e;
          if (col <= row) S[row * LDS + col] -= acc[e];
        }
      }
      __syncthreads();
    }
    // the off-diagonal blocks of L (the diagonal blocks went out from warp 0's registers)
    for (int e = tid; e < NB * NB; e += LEAF_THREADS) {
      const int r = e % NB, c = e / NB;
      if ((r >> 5) == (c >> 5)) continue;
      Ab[r + (long long)c * ld] = (r > c) ? S[r * LDS + c] : 0.0;
    }
  } else {   // inverse only: T_J of the four diagonal blocks, one warp each
    double tc[LB];
    if (warp < NB / LB) warp_inverse32(S, warp * LB, tc, lane);
    __syncthreads();
    if (warp < NB / LB) {
#pragma unroll
      for (int i = 0; i < LB; ++i) S[(warp * LB + i) * LDS + warp * LB + lane] = tc[i];
    }
  }
  __syncthreads();
  // ---- inverse phases (S diagonal blocks = T_J, strictly upper part of S = 0) ----
  // (a) W_b = L_IJ T_J for (I, J) = (1, 0), (3, 2): T_J[k][c] = 0 for k < c
  for (int job = warp; job < 32; job += LEAF_WARPS) {
    const int b = job >> 4, rt = (job >> 2) & 3, ct = job & 3;
    const int I = 2 * b + 1, J = 2 * b;
    double acc[2];
    tile8<false>(acc, S + J * LB, LDS, I * LB + 8 * rt, S + J * LB * LDS + J * LB, LDS, 8 * ct,
                 8 * ct, LB, lane);
#pragma unroll
    for (int e = 0; e < 2; ++e) W[(b * LB + 8 * rt + g) * WLD + 8 * ct + 2 * t4 + e] = acc[e];
  }
  __syncthreads();
  // (b) X_IJ = -T_I W_b (T_I[r][k] = 0 for k > r), over L_IJ
  for (int job = warp; job < 32; job += LEAF_WARPS) {
    const int b = job >> 4, rt = (job >> 2) & 3, ct = job & 3;
    const int I = 2 * b + 1, J = 2 * b;
    double acc[2];
    tile8<false>(acc, S + I * LB, LDS, I * LB + 8 * rt, W + b * LB * WLD, WLD, 8 * ct, 0,
                 8 * rt + 8, lane);
#pragma unroll
    for (int e = 0; e < 2; ++e) S[(I * LB + 8 * rt + g) * LDS + J * LB + 8 * ct + 2 * t4 + e] = -acc[e];
  }
  __syncthreads();
  // (c) W = L[64:, :64] X_A (X_A = S[:64, :64], lower)
  for (int job = warp; job < 64; job += LEAF_WARPS) {
    const int rt = job >> 3, ct = job & 7;
    double acc[2];
    tile8<false>(acc, S, LDS, 64 + 8 * rt, S, LDS, 8 * ct, 8 * ct, 64, lane);
#pragma unroll
    for (int e = 0; e < 2; ++e) W[(8 * rt + g) * WLD + 8 * ct + 2 * t4 + e] = acc[e];
  }
  __syncthreads();
  // (d) X[64:, :64] = -X_C W (X_C = S[64:, 64:], lower), over L[64:, :64]
  for (int job = warp; job < 64; job += LEAF_WARPS) {
    const int rt = job >> 3, ct = job & 7;
    double acc[2];
    tile8<false>(acc, S + 64, LDS, 64 + 8 * rt, W, WLD, 8 * ct, 0, 8 * rt + 8, lane);
#pragma unroll
    for (int e = 0; e < 2; ++e) S[(64 + 8 * rt + g) * LDS + 8 * ct + 2 * t4 + e] = -acc[e];
  }
  __syncthreads();
  double* Db = Dinv + k0 + (panel ? 0ll : (long long)k0 * ldi);
  for (int e = tid; e < NB * NB; e += LEAF_THREADS) {
    const int r = e % NB, c = e / NB;
    Db[r + (long long)c * ldi] = (r >= c) ? S[r * LDS + c] : 0.0;
  }
}


int grid_for(long long total) {
  long long g = (total + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

// The large factorisation GEMMs go to the int8 tensor cores (ozaki_i8.cu) unless
// GG_FACTOR_OZAKI=0; below OZ_MIN_DIM in any dimension the DMMA kernel is used.
constexpr int OZ_MIN_DIM = 512;
bool use_ozaki() {
  const char* v = getenv("GG_FACTOR_OZAKI");
  return v == nullptr ? OZAKI_DEFAULT : v[0] != '0';
}
bool oz_shape(int M, int N, int K) {
  return M >= OZ_MIN_DIM && N >= OZ_MIN_DIM && K >= OZ_MIN_DIM;
}

// Ozaki workspace of the trtri recursion on [lo, hi) (its two GEMMs per level)
size_t trtri_oz_bytes(int lo, int hi) {
  const int nblk = (hi - lo) / NB;
  if (nblk < 2) return 0;
  const int mid = lo + (nblk / 2) * NB;
  size_t b = trtri_oz_bytes(lo, mid);
  const size_t b2 = trtri_oz_bytes(mid, hi);
  if (b2 > b) b = b2;
  if (oz_shape(hi - mid, mid - lo, mid - lo)) {
    const size_t g1 = ozaki_ws_bytes(hi - mid, mid - lo, mid - lo, false);
    const size_t g2 = ozaki_ws_bytes(hi - mid, mid - lo, hi - mid, false);
    if (g1 > b) b = g1;
    if (g2 > b) b = g2;
  }
  return b;
}

// Off-diagonal blocks of Linv for the block range [lo, hi) (diagonal blocks already set).
int trtri_offdiag(int lo, int hi, const double* L, double* Linv, long long ldp, double* T,
                  long long ldt, void* oz, size_t oz_bytes, const int* abort_flag,
                  cudaStream_t s) {
  const int nblk = (hi - lo) / NB;
  if (nblk < 2) return GG_OK;
  const int mid = lo + (nblk / 2) * NB;
  int rc = trtri_offdiag(lo, mid, L, Linv, ldp, T, ldt, oz, oz_bytes, abort_flag, s);
  if (rc != GG_OK) return rc;
  rc = trtri_offdiag(mid, hi, L, Linv, ldp, T, ldt, oz, oz_bytes, abort_flag, s);
  if (rc != GG_OK) return rc;
  if (oz != nullptr && oz_shape(hi - mid, mid - lo, mid - lo)) {
    // T = L[mid:hi, lo:mid] Linv[lo:mid, lo:mid]  (B~(j,k) = Linv[lo+k, lo+j], zero for k < j)
    rc = ozaki_gemm_run(hi - mid, mid - lo, mid - lo, L + mid + (long long)lo * ldp, 1, ldp,
                        Linv + lo + (long long)lo * ldp, ldp, 1, T, ldt, 1.0, 0.0, GEMM_B_LOWER,
                        oz, oz_bytes, abort_flag, s);
    if (rc != GG_OK) return rc;
    // Linv[mid:hi, lo:mid] = -Linv[mid:hi, mid:hi] T  (A~ lower triangular, B~(j,k) = T[k, j])
    return ozaki_gemm_run(hi - mid, mid - lo, hi - mid, Linv + mid + (long long)mid * ldp, 1, ldp,
                          T, ldt, 1, Linv + mid + (long long)lo * ldp, ldp, -1.0, 0.0,
                          GEMM_A_LOWER, oz, oz_bytes, abort_flag, s);
  }
  // T = L[mid:hi, lo:mid] * Linv[lo:mid, lo:mid]      (op(B) lower triangular)
  GemmArgs g1{};
  g1.M = hi - mid; g1.N = mid - lo; g1.K = mid - lo;
  g1.A = L + mid + (long long)lo * ldp; g1.lda = ldp;
  g1.B = Linv + lo + (long long)lo * ldp; g1.ldb = ldp;
  g1.C = T; g1.ldc = ldt;
  g1.alpha = 1.0; g1.beta = 0.0; g1.flags = GEMM_B_LOWER; g1.abort_flag = abort_flag;
  rc = launch_dgemm(g1, false, s);
  if (rc != GG_OK) return rc;
  // Linv[mid:hi, lo:mid] = -Linv[mid:hi, mid:hi] * T   (A lower triangular)
  GemmArgs g2{};
  g2.M = hi - mid; g2.N = mid - lo; g2.K = hi - mid;
  g2.A = Linv + mid + (long long)mid * ldp; g2.lda = ldp;
  g2.B = T; g2.ldb = ldt;
  g2.C = Linv + mid + (long long)lo * ldp; g2.ldc = ldp;
  g2.alpha = -1.0; g2.beta = 0.0; g2.flags = GEMM_A_LOWER; g2.abort_flag = abort_flag;
  return launch_dgemm(g2, false, s);
}

void trtri_T_dims(int np, long long* rows, long long* cols) {
  const int nblk = np / NB;
  if (nblk < 2) { *rows = 0; *cols = 0; return; }
  *cols = (long long)(nblk / 2) * NB;
  *rows = (long long)(nblk - nblk / 2) * NB;
}


// Workspace: [header][panel / trtri T][Ozaki slices]
size_t t_region_bytes(int np) {
  long long r, c;
  trtri_T_dims(np, &r, &c);
  return ((size_t)(r * c) * sizeof(double) + 255) & ~size_t(255);
}
size_t oz_region_bytes(int np, bool factor) {
  size_t b = trtri_oz_bytes(0, np);
  if (factor) {   // the trailing SYRKs: largest at the first outer block
    const int rem = np - OUTER;
    if (rem > 0 && oz_shape(rem, rem, OUTER)) {
      const size_t sy = ozaki_ws_bytes(rem, rem, OUTER, true);
      if (sy > b) b = sy;
    }
  }
  return b;
}

}  // namespace

size_t trtri_ws_bytes(int n) {
  const int np = pad_rows(n);
  return HDR_BYTES + t_region_bytes(np) + oz_region_bytes(np, false);
}

size_t potrf_ws_bytes(int n) {
  const int np = pad_rows(n);
  size_t panel = ((size_t)np * NB * sizeof(double) + 255) & ~size_t(255);
  const size_t tri = t_region_bytes(np);
  if (tri > panel) panel = tri;
  return HDR_BYTES + panel + oz_region_bytes(np, true);
}

namespace {
size_t p_region_bytes(int np) {
  size_t panel = ((size_t)np * NB * sizeof(double) + 255) & ~size_t(255);
  const size_t tri = t_region_bytes(np);
  return tri > panel ? tri : panel;
}
}  // namespace

int potrf_run(int n, const double* M, int ldm, int m_row_major, double* L, double* Linv, int ldp, void* work,
              int* info_host, cudaStream_t s) {
  if (n < 1 || M == nullptr || L == nullptr || Linv == nullptr || work == nullptr ||
      info_host == nullptr) {
    set_error("potrf: null pointer or n < 1");
    return GG_EARG;
  }
  const int np = pad_rows(n);
  if (ldm < n || ldp < np) {
    set_error("potrf: leading dimension too small (ldm >= n, ldp >= gg_pad(n))");
    return GG_EDIM;
  }
  info_host[0] = -1;
  info_host[1] = 0;
  PotrfHeader* hdr = static_cast<PotrfHeader*>(work);
  double* P = reinterpret_cast<double*>(static_cast<char*>(work) + HDR_BYTES);
  const size_t oz_bytes = use_ozaki() ? oz_region_bytes(np, true) : 0;
  void* oz = oz_bytes ? static_cast<char*>(work) + HDR_BYTES + p_region_bytes(np) : nullptr;
  GG_CUDA_TRY(cudaMemsetAsync(hdr, 0, sizeof(int) * 2, s));
  GG_CUDA_TRY(cudaMemsetAsync(&hdr->nonfinite, 0xff, sizeof(unsigned long long), s));
  const long long rs = m_row_major ? ldm : 1, cs = m_row_major ? 1 : ldm;
  init_factor_tiled_kernel<<<dim3(np / 32, np / 32), 256, 0, s>>>(n, np, M, rs, cs, L, Linv, ldp,
                                                                  &hdr->nonfinite);
  GG_LAUNCH_CHECK("init_factor_tiled_kernel");
  GG_CUDA_TRY(cudaFuncSetAttribute(leaf_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)LEAF_SMEM));
  // optional phase timing (GG_POTRF_TIMING=1): leaf / panel / trailing / inverse, to stderr
  const bool timing = getenv("GG_POTRF_TIMING") != nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  float t_leaf = 0.f, t_pan = 0.f, t_upd = 0.f, t_inv = 0.f;
  if (timing)
    for (auto& e : ev) cudaEventCreate(&e);
  auto lap = [&](float& acc, cudaEvent_t a, cudaEvent_t b) {
    if (!timing) return;
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    acc += ms;
  };
  // Two-level right-looking blocking: outer block columns of OUTER (= 8 leaves); inside one,
  // leaf + panel + an update restricted to the outer block's columns; after it, one trailing
  // SYRK of depth OUTER (8x the arithmetic intensity of a depth-128 update; 1024 measured best
  // between 256 and 4096 at n = 1e4 and 4e4).
  for (int K0 = 0; K0 < np; K0 += OUTER) {
    const int w = (np - K0 < OUTER) ? (np - K0) : OUTER;
    for (int k = K0; k < K0 + w; k += NB) {
      if (timing) cudaEventRecord(ev[0], s);
      leaf_kernel<true><<<1, LEAF_THREADS, LEAF_SMEM, s>>>(L, ldp, Linv, ldp, k, &hdr->info);
      GG_LAUNCH_CHECK("potrf leaf_kernel");
      lap(t_leaf, ev[0], ev[1]);
      const int rem = np - k - NB;          // rows below this leaf
      if (rem <= 0) break;
      const int rem_in = K0 + w - k - NB;   // columns of the outer block right of this leaf
      // P = A21 Dinv^T (all rows below), written back into L's column block
      GemmArgs pan{};
      pan.M = rem; pan.N = NB; pan.K = NB;
      pan.A = L + (k + NB) + (long long)k * ldp; pan.lda = ldp;
      pan.B = Linv + k + (long long)k * ldp; pan.ldb = ldp;
      pan.C = P; pan.ldc = np;
      pan.alpha = 1.0; pan.beta = 0.0; pan.flags = 0; pan.abort_flag = &hdr->info;
      int rc = launch_dgemm(pan, true, s);
      if (rc != GG_OK) return rc;
      GG_CUDA_TRY(cudaMemcpy2DAsync(L + (k + NB) + (long long)k * ldp,
                                    (size_t)ldp * sizeof(double), P, (size_t)np * sizeof(double),
                                    (size_t)rem * sizeof(double), NB, cudaMemcpyDeviceToDevice, s));
      lap(t_pan, ev[1], ev[2]);
      if (rem_in > 0) {
        // update only the outer block's remaining columns: A[k+NB:, k+NB:K0+w] -= P P[:rem_in]^T
        GemmArgs upd{};
        upd.M = rem; upd.N = rem_in; upd.K = NB;
        upd.A = P; upd.lda = np;
        upd.B = P; upd.ldb = np;
        upd.C = L + (k + NB) + (long long)(k + NB) * ldp; upd.ldc = ldp;
        upd.alpha = -1.0; upd.beta = 1.0; upd.flags = GEMM_C_LOWER; upd.abort_flag = &hdr->info;
        rc = launch_dgemm(upd, true, s);
        if (rc != GG_OK) return rc;
      }
      lap(t_upd, ev[2], ev[3]);
    }
    const int rem = np - K0 - w;
    if (rem <= 0) break;
    if (timing) cudaEventRecord(ev[2], s);
    // trailing SYRK of depth w: A22 -= L21 L21^T, L21 = L[K0+w:, K0:K0+w] (read in place;
    // disjoint from the updated region), lower tiles only
    int rc;
    if (oz != nullptr && oz_shape(rem, rem, w)) {
      rc = ozaki_gemm_run(rem, rem, w, L + (K0 + w) + (long long)K0 * ldp, 1, ldp, nullptr, 0, 0,
                          L + (K0 + w) + (long long)(K0 + w) * ldp, ldp, -1.0, 1.0, GEMM_C_LOWER,
                          oz, oz_bytes, &hdr->info, s);
    } else {
      GemmArgs upd{};
      upd.M = rem; upd.N = rem; upd.K = w;
      upd.A = L + (K0 + w) + (long long)K0 * ldp; upd.lda = ldp;
      upd.B = L + (K0 + w) + (long long)K0 * ldp; upd.ldb = ldp;
      upd.C = L + (K0 + w) + (long long)(K0 + w) * ldp; upd.ldc = ldp;
      upd.alpha = -1.0; upd.beta = 1.0; upd.flags = GEMM_C_LOWER; upd.abort_flag = &hdr->info;
      rc = launch_dgemm(upd, true, s);
    }
    if (rc != GG_OK) return rc;
    lap(t_upd, ev[2], ev[3]);
  }
  if (timing) cudaEventRecord(ev[0], s);
  long long tr, tc;
  trtri_T_dims(np, &tr, &tc);
  int rc = trtri_offdiag(0, np, L, Linv, ldp, P, tr > 0 ? tr : 1, oz, oz_bytes, &hdr->info, s);
  if (rc != GG_OK) return rc;
  lap(t_inv, ev[0], ev[1]);
  if (timing) {
    fprintf(stderr, "[gg potrf n=%d] leaf %.2f ms, panel %.2f ms, trailing %.2f ms, inverse %.2f ms\n",
            n, t_leaf, t_pan, t_upd, t_inv);
    for (auto& e : ev) cudaEventDestroy(e);
  }
  PotrfHeader h{};
  GG_CUDA_TRY(cudaMemcpyAsync(&h, hdr, sizeof(PotrfHeader), cudaMemcpyDeviceToHost, s));
  GG_CUDA_TRY(cudaStreamSynchronize(s));
  if (h.nonfinite != ULLONG_MAX) {
    info_host[0] = (int)(h.nonfinite / (unsigned long long)n);
    info_host[1] = 1;
    set_error("non-finite entry in covariance");
    return GG_ENOTPD;
  }
  if (h.info != 0) {
    info_host[0] = h.info - 1;
    set_error("matrix not positive definite");
    return GG_ENOTPD;
  }
  return GG_OK;
}

int trtri_run(int n, const double* L, int ldl, double* Linv, int ldp, void* work, cudaStream_t s) {
  if (n < 1 || L == nullptr || Linv == nullptr || work == nullptr) {
    set_error("trtri: null pointer or n < 1");
    return GG_EARG;
  }
  const int np = pad_rows(n);
  if (ldl < np || ldp < np) {
    set_error("trtri: leading dimension too small (>= gg_pad(n))");
    return GG_EDIM;
  }
  if (ldl != ldp) {
    set_error("trtri: ldl must equal ldp");
    return GG_EDIM;
  }
  double* T = reinterpret_cast<double*>(static_cast<char*>(work) + HDR_BYTES);
  zero_square_kernel<<<grid_for((long long)np * np), 256, 0, s>>>(np, Linv, ldp);
  GG_LAUNCH_CHECK("zero_square_kernel");
  GG_CUDA_TRY(cudaFuncSetAttribute(leaf_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)LEAF_SMEM));
  // leaf_kernel<false> only reads L; the const_cast never results in a write.
  leaf_kernel<false><<<np / NB, LEAF_THREADS, LEAF_SMEM, s>>>(const_cast<double*>(L), ldl, Linv,
                                                               ldp, 0, nullptr);
  GG_LAUNCH_CHECK("trtri leaf_kernel");
  long long tr, tc;
  trtri_T_dims(np, &tr, &tc);
  const size_t oz_bytes = use_ozaki() ? oz_region_bytes(np, false) : 0;
  void* oz = oz_bytes ? static_cast<char*>(work) + HDR_BYTES + t_region_bytes(np) : nullptr;
  return trtri_offdiag(0, np, L, Linv, ldp, T, tr > 0 ? tr : 1, oz, oz_bytes, nullptr, s);
}

// Blocked forward substitution X = L^-1 B (kernel.trsolve_lower for an arbitrary L): the inverses
// of all 128 x 128 diagonal blocks in one leaf launch (an np x 128 panel), then per block column J
//   X_J = Dinv_J B_J                 (DMMA GEMM, 128 x nrhs x 128)
//   B_{J+1:} -= L_{J+1:, J} X_J     (DMMA GEMM, rows below x nrhs x 128)
// O(n^2 nrhs) work, backward-stable like dtrsm's blocked form (no O(n^3) full inverse).  X may
// alias B (the right-hand side is consumed in place when it does).
size_t trsm_blocked_ws_bytes(int n, int nrhs) {
  const size_t np = (size_t)pad_rows(n);
  return np * NB * sizeof(double) + (size_t)NB * (size_t)(nrhs > 0 ? nrhs : 1) * sizeof(double) +
         256;
}

int trsm_blocked_run(int n, int nrhs, const double* L, int ldl, const double* B, int ldb,
                     double* X, int ldx, void* work, cudaStream_t s) {
  const int np = pad_rows(n);
  if (ldl < np || ldb < np || ldx < np) {
    set_error("trsm_blocked: leading dimensions must be >= gg_pad(n)");
    return GG_EDIM;
  }
  if (nrhs <= 0) return GG_OK;
  double* D = static_cast<double*>(work);                      // np x 128, ld np
  double* Y = D + (size_t)np * NB;                             // 128 x nrhs, ld 128
  GG_CUDA_TRY(cudaFuncSetAttribute(leaf_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)LEAF_SMEM));
  leaf_kernel<false><<<np / NB, LEAF_THREADS, LEAF_SMEM, s>>>(const_cast<double*>(L), ldl, D,
                                                               np, 0, nullptr, 1);
  GG_LAUNCH_CHECK("trsm_blocked leaf_kernel");
  if (X != B)
    GG_CUDA_TRY(cudaMemcpy2DAsync(X, (size_t)ldx * sizeof(double), B, (size_t)ldb * sizeof(double),
                                  (size_t)np * sizeof(double), nrhs, cudaMemcpyDeviceToDevice, s));
  for (int J = 0; J < np; J += NB) {
    GemmArgs d{};
    d.M = NB; d.N = nrhs; d.K = NB;
    d.A = D + J; d.lda = np;
    d.B = X + J; d.ldb = ldx;
    d.C = Y; d.ldc = NB;
    d.alpha = 1.0; d.beta = 0.0; d.flags = GEMM_A_LOWER; d.abort_flag = nullptr;
    int rc = launch_dgemm(d, false, s);
    if (rc != GG_OK) return rc;
    GG_CUDA_TRY(cudaMemcpy2DAsync(X + J, (size_t)ldx * sizeof(double), Y, NB * sizeof(double),
                                  NB * sizeof(double), nrhs, cudaMemcpyDeviceToDevice, s));
    const int rem = np - J - NB;
    if (rem <= 0) break;
    GemmArgs u{};
    u.M = rem; u.N = nrhs; u.K = NB;
    u.A = L + (J + NB) + (long long)J * ldl; u.lda = ldl;
    u.B = X + J; u.ldb = ldx;
    u.C = X + J + NB; u.ldc = ldx;
    u.alpha = -1.0; u.beta = 1.0; u.flags = 0; u.abort_flag = nullptr;
    rc = launch_dgemm(u, false, s);
    if (rc != GG_OK) return rc;
  }
  return GG_OK;
}

}  // namespace gg
