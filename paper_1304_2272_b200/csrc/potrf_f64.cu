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
#ifndef GG_OUTER
#define GG_OUTER (8 * 128)
#endif
constexpr int OUTER = GG_OUTER;   // outer block width of the two-level Cholesky
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
// Column j is broadcast through shared memory (sm: 2 x 32 doubles, 16-byte aligned, alternating
// by j): one store per lane, then the pivot and the column pairs are broadcast LDS.128 reads --
// r02 shuffled every column entry (two SHFLs per double, 62 per pivot at j = 0: ~410 cycles per
// pivot).  Every lane scales the broadcast unscaled entry itself (lc = u_c rs), the same DMUL the
// owning lane applies to its own entry, so the factor is bitwise that of the shuffle form.
__device__ __forceinline__ int warp_factor32(double (&r)[LB], int lane, double* sm) {
  int fail = -1;
#pragma unroll
  for (int j = 0; j < LB; ++j) {
    double* col = sm + (j & 1) * LB;
    col[lane] = r[j];                            // unscaled column j
    __syncwarp();
    double d = col[j];
    if (fail < 0 && !(d > 0.0)) fail = j;        // uniform: every lane sees the same d
    if (fail >= 0) d = 1.0;                      // keep the arithmetic finite past a failure
    // the scale must be the rounded reciprocal of the stored pivot (dpotf2): rsqrt(d) instead
    // measured 10x larger GLS errors on AR(1) covariances (rho = 0.999: 5.3e-10 vs 5.1e-11), and
    // rsqrt(d) with piv = RN(1/rs) 4x larger (and no faster)
    const double piv = __dsqrt_rn(d), rs = __drcp_rn(piv);   // = sqrt(d), 1.0 / piv
    if (lane == j) r[j] = piv;
    else if (lane > j) r[j] *= rs;
#pragma unroll
    for (int c = 0; c < LB; c += 2) {   // constant bounds: fully unrolled, r[] stays in registers
      if (c + 1 > j) {
        const double2 u = *reinterpret_cast<const double2*>(col + c);
        if (c > j) {
          const double lc = u.x * rs;
          if (lane >= c) r[c] -= r[j] * lc;
        }
        const double lc1 = u.y * rs;
        if (lane >= c + 1) r[c + 1] -= r[j] * lc1;
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

#ifdef GG_LEAF_PROFILE
__device__ long long g_leaf_ts[64];
#endif
template <bool FACTOR>
__global__ void __launch_bounds__(LEAF_THREADS, 1) leaf_kernel(double* A, long long ld,
                                                               double* Dinv, long long ldi, int k0,
                                                               int* info, int panel = 0) {
  extern __shared__ double lsm[];
#ifdef GG_LEAF_PROFILE   // measurement builds: clock64 at every barrier of the factoring leaf
  int tsi = 0;
  if (FACTOR && threadIdx.x == 0) g_leaf_ts[tsi++] = clock64();
#define LEAF_TS() do { if (FACTOR && threadIdx.x == 0 && tsi < 64) g_leaf_ts[tsi++] = clock64(); } while (0)
#else
#define LEAF_TS() do { } while (0)
#endif
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
  LEAF_TS();
  if (FACTOR) {
    // Look-ahead inside the leaf: the trailing update of panel J-1 is split -- warps 0-3 update the
    // diagonal block J (10 lower 8 x 8 tiles, named barrier 1) and warp 0 goes straight on to
    // factor and invert it, while warps 1-11 update the rest of the trailing region; one barrier
    // joins them before panel J.
    // (r02: the trailing updates ran between barriers, 9k of 110k cycles on the critical path.)
    for (int J = 0; J < NB / LB; ++J) {
      const int j0 = J * LB;
      if (J > 0 && warp < 4) {   // S_JJ -= L_J,J-1 L_J,J-1^T: 10 lower 8 x 8 tiles on warps 0-3
        for (int tt = warp; tt < 10; tt += 4) {
          int rt = 0;
          while ((rt + 1) * (rt + 2) / 2 <= tt) ++rt;
          const int ct = tt - rt * (rt + 1) / 2;
          const int r0 = j0 + 8 * rt, c0 = j0 + 8 * ct;
          double acc[2];
          tile8<true>(acc, S + j0 - LB, LDS, r0, S + j0 - LB, LDS, c0, 0, LB, lane);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int row = r0 + g, col = c0 + 2 * t4 + e;
            if (col <= row) S[row * LDS + col] -= acc[e];
          }
        }
        asm volatile("bar.sync 1, 128;\n" ::: "memory");   // warps 0-3 only
      }
      if (warp == 0) {
        double r[LB];
#pragma unroll
        for (int c = 0; c < LB; ++c) r[c] = S[(j0 + lane) * LDS + j0 + c];
        const int f = warp_factor32(r, lane, W);   // W: scratch until the inverse phases
        LEAF_TS();
        if (f >= 0) {
          if (lane == 0) *fail = j0 + f;
        } else {
#pragma unroll
          for (int c = 0; c < LB; ++c) {
            S[(j0 + lane) * LDS + j0 + c] = r[c];
            Ab[(j0 + lane) + (long long)(j0 + c) * ld] = (lane >= c) ? r[c] : 0.0;
          }
          __syncwarp();
          LEAF_TS();
          double tc[LB];
          warp_inverse32(S, j0, tc, lane);
          __syncwarp();
          LEAF_TS();
#pragma unroll
          for (int i = 0; i < LB; ++i) S[(j0 + i) * LDS + j0 + lane] = tc[i];
        }
      } else if (J > 0) {
        // the rest of panel J-1's trailing update (warps 1-11): lower 8 x 8 tiles of rows /
        // columns [j0, 128) outside the diagonal block J
        const int m = (NB - j0) / 8;
        for (int tt = warp - 1; tt < m * (m + 1) / 2; tt += LEAF_WARPS - 1) {
          int rt = 0;
          while ((rt + 1) * (rt + 2) / 2 <= tt) ++rt;
          const int ct = tt - rt * (rt + 1) / 2;
          if (rt < LB / 8) continue;   // diagonal block J: done above
          const int r0 = j0 + 8 * rt, c0 = j0 + 8 * ct;
          double acc[2];
          tile8<true>(acc, S + j0 - LB, LDS, r0, S + j0 - LB, LDS, c0, 0, LB, lane);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int row = r0 + g, col = c0 + 2 * t4 + e;
            if (col <= row) S[row * LDS + col] -= acc[e];
          }
        }
      }
      __syncthreads();
      LEAF_TS();
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
      LEAF_TS();
    }
    // the off-diagonal blocks of L (the diagonal blocks went out from warp 0's registers); no
    // barrier before inverse phase (a), which only reads S as well
    for (int e = tid; e < NB * NB; e += LEAF_THREADS) {
      const int r = e % NB, c = e / NB;
      if ((r >> 5) == (c >> 5)) continue;
      Ab[r + (long long)c * ld] = (r > c) ? S[r * LDS + c] : 0.0;
    }
  } else {   // inverse only: T_J of the four diagonal blocks, one warp each
    double tc[LB];
    if (warp < NB / LB) warp_inverse32(S, warp * LB, tc, lane);
    __syncthreads();
    LEAF_TS();
    if (warp < NB / LB) {
#pragma unroll
      for (int i = 0; i < LB; ++i) S[(warp * LB + i) * LDS + warp * LB + lane] = tc[i];
    }
    __syncthreads();
  }
  LEAF_TS();
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
  LEAF_TS();
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
  LEAF_TS();
  // (c) W = L[64:, :64] X_A (X_A = S[:64, :64], lower)
  for (int job = warp; job < 64; job += LEAF_WARPS) {
    const int rt = job >> 3, ct = job & 7;
    double acc[2];
    tile8<false>(acc, S, LDS, 64 + 8 * rt, S, LDS, 8 * ct, 8 * ct, 64, lane);
#pragma unroll
    for (int e = 0; e < 2; ++e) W[(8 * rt + g) * WLD + 8 * ct + 2 * t4 + e] = acc[e];
  }
  __syncthreads();
  LEAF_TS();
  // (d) X[64:, :64] = -X_C W (X_C = S[64:, 64:], lower), over L[64:, :64]
  for (int job = warp; job < 64; job += LEAF_WARPS) {
    const int rt = job >> 3, ct = job & 7;
    double acc[2];
    tile8<false>(acc, S + 64, LDS, 64 + 8 * rt, W, WLD, 8 * ct, 0, 8 * rt + 8, lane);
#pragma unroll
    for (int e = 0; e < 2; ++e) S[(64 + 8 * rt + g) * LDS + 8 * ct + 2 * t4 + e] = -acc[e];
  }
  __syncthreads();
  LEAF_TS();
  double* Db = Dinv + k0 + (panel ? 0ll : (long long)k0 * ldi);
  for (int e = tid; e < NB * NB; e += LEAF_THREADS) {
    const int r = e % NB, c = e / NB;
    Db[r + (long long)c * ldi] = (r >= c) ? S[r * LDS + c] : 0.0;
  }
  __syncthreads();
  LEAF_TS();
#undef LEAF_TS
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

// ---- off-diagonal blocks of Linv, bottom-up ----------------------------------------------------
// Level b = 128 2^j combines pairs of already inverted diagonal ranges [lo, mid = lo + b) and
// [mid, hi = min(lo + 2b, np)) (lo = 2b i):
//     T = L[mid:hi, lo:mid] Linv[lo:mid, lo:mid],   Linv[mid:hi, lo:mid] = -Linv[mid:hi, mid:hi] T.
// The groups of a level are independent: the full ones are ONE strided-batched DMMA launch per
// product (r02: a depth-first recursion issued ~150 launches of 1-6 CTAs at n = 1e4, 13 ms); the
// partial last group is its own launch; levels with b >= OZ_TRTRI_MIN go to the Ozaki GEMM per
// group (large products, where the int8 tensor cores' 2x beats DMMA).  T of group i sits at
// T + i b^2 with ld = its row count.
constexpr int OZ_TRTRI_MIN = 4096;

struct TrtriLevel {
  int b, nfull, mlast;   // half width, full groups, rows of the partial last group (0: none)
};
inline TrtriLevel trtri_level(int np, int b) {
  TrtriLevel l{b, 0, 0};
  for (int lo = 0; lo + b < np; lo += 2 * b) {
    const int m = (lo + 2 * b <= np) ? b : np - lo - b;
    if (m == b) ++l.nfull;
    else l.mlast = m;
  }
  return l;
}
size_t trtri_T_doubles(int np) {
  size_t mx = 0;
  for (int b = NB; b < np; b *= 2) {
    const TrtriLevel l = trtri_level(np, b);
    const size_t d = (size_t)l.nfull * b * b + (size_t)l.mlast * b;
    if (d > mx) mx = d;
  }
  return mx;
}
size_t trtri_oz_bytes(int np) {
  size_t mx = 0;
  for (int b = OZ_TRTRI_MIN; b < np; b *= 2) {
    const TrtriLevel l = trtri_level(np, b);
    for (int m : {l.nfull ? b : 0, l.mlast}) {
      if (m == 0 || !oz_shape(m, b, b)) continue;
      const size_t g1 = ozaki_ws_bytes(m, b, b, false), g2 = ozaki_ws_bytes(m, b, m, false);
      if (g1 > mx) mx = g1;
      if (g2 > mx) mx = g2;
    }
  }
  return mx;
}

// the two products of `count` consecutive groups of level b starting at group g0, M rows each
int trtri_groups(int b, int g0, int count, int M, const double* L, double* Linv, long long ldp,
                 double* T, void* oz, size_t oz_bytes, const int* abort_flag, cudaStream_t s) {
  const long long step = 2ll * b * (1 + ldp);              // next group along the diagonal
  const long long lo = 2ll * b * g0, mid = lo + b;
  double* Tg = T + (size_t)g0 * b * b;
  if (oz != nullptr && b >= OZ_TRTRI_MIN && oz_shape(M, b, b)) {
    for (int i = 0; i < count; ++i) {
      const long long o = i * step;
      double* Ti = Tg + (size_t)i * b * b;
      int rc = ozaki_gemm_run(M, b, b, L + mid + lo * ldp + o, 1, ldp, Linv + lo + lo * ldp + o,
                              ldp, 1, Ti, M, 1.0, 0.0, GEMM_B_LOWER, oz, oz_bytes, abort_flag, s);
      if (rc != GG_OK) return rc;
      rc = ozaki_gemm_run(M, b, M, Linv + mid + mid * ldp + o, 1, ldp, Ti, M, 1,
                          Linv + mid + lo * ldp + o, ldp, -1.0, 0.0, GEMM_A_LOWER, oz, oz_bytes,
                          abort_flag, s);
      if (rc != GG_OK) return rc;
    }
    return GG_OK;
  }
  GemmArgs g1{};   // T = L[mid:hi, lo:mid] Linv[lo:mid, lo:mid]   (op(B) lower triangular)
  g1.M = M; g1.N = b; g1.K = b;
  g1.A = L + mid + lo * ldp; g1.lda = ldp;
  g1.B = Linv + lo + lo * ldp; g1.ldb = ldp;
  g1.C = Tg; g1.ldc = M;
  g1.alpha = 1.0; g1.beta = 0.0; g1.flags = GEMM_B_LOWER; g1.abort_flag = abort_flag;
  g1.batch = count; g1.sA = step; g1.sB = step; g1.sC = (long long)b * b;
  int rc = launch_dgemm(g1, false, s);
  if (rc != GG_OK) return rc;
  GemmArgs g2{};   // Linv[mid:hi, lo:mid] = -Linv[mid:hi, mid:hi] T   (A lower triangular)
  g2.M = M; g2.N = b; g2.K = M;
  g2.A = Linv + mid + mid * ldp; g2.lda = ldp;
  g2.B = Tg; g2.ldb = M;
  g2.C = Linv + mid + lo * ldp; g2.ldc = ldp;
  g2.alpha = -1.0; g2.beta = 0.0; g2.flags = GEMM_A_LOWER; g2.abort_flag = abort_flag;
  g2.batch = count; g2.sA = step; g2.sB = (long long)b * b; g2.sC = step;
  return launch_dgemm(g2, false, s);
}

// Off-diagonal blocks of Linv (its 128 x 128 diagonal blocks already set).
int trtri_offdiag(int np, const double* L, double* Linv, long long ldp, double* T, void* oz,
                  size_t oz_bytes, const int* abort_flag, cudaStream_t s) {
  for (int b = NB; b < np; b *= 2) {
    const TrtriLevel l = trtri_level(np, b);
    int rc = GG_OK;
    if (l.nfull > 0)
      rc = trtri_groups(b, 0, l.nfull, b, L, Linv, ldp, T, oz, oz_bytes, abort_flag, s);
    if (rc == GG_OK && l.mlast > 0)
      rc = trtri_groups(b, l.nfull, 1, l.mlast, L, Linv, ldp, T, oz, oz_bytes, abort_flag, s);
    if (rc != GG_OK) return rc;
  }
  return GG_OK;
}

// Workspace: [header][panels (2 x np x 128, double-buffered for the look-ahead) / trtri T]
//            [Ozaki slices]
size_t t_region_bytes(int np) {
  return (trtri_T_doubles(np) * sizeof(double) + 255) & ~size_t(255);
}
// Trailing-update aggregation: the far columns' SYRK runs once per `syrk_agg()` outer blocks with
// the deferred panels stacked along k (depth agg OUTER); the outer blocks in between update only
// the next outer block's columns.  Same arithmetic, 1/agg the passes over the trailing matrix
// (each pass re-reads and re-writes C and pays the per-tile epilogue).  Tuning knob GG_SYRK_AGG.
int syrk_agg() {
  const char* v = getenv("GG_SYRK_AGG");
  const int a = v ? atoi(v) : 1;
  return a < 1 ? 1 : (a > 8 ? 8 : a);
}
// the trailing update after outer block K0 (width w): columns [K0+w, K0+w+ncols) of all rows
// below, from the panels [dstart, K0+w) -- returns false when there is none
struct TrailingUpdate {
  int rem, ncols, kd;
  bool full;
};
bool trailing_update(int np, int K0, int w, int dstart, int agg, TrailingUpdate* t) {
  t->rem = np - K0 - w;
  if (t->rem <= 0) return false;
  t->full = ((K0 / OUTER + 1) % agg == 0) || t->rem <= OUTER;
  t->ncols = t->full ? t->rem : OUTER;
  t->kd = K0 + w - dstart;
  return true;
}

size_t oz_region_bytes(int np, bool factor) {
  size_t b = trtri_oz_bytes(np);
  if (factor) {   // the trailing SYRKs, as potrf_run issues them
    const int agg = syrk_agg();
    int dstart = 0;
    TrailingUpdate t;
    for (int K0 = 0; K0 < np; K0 += OUTER) {
      const int w = (np - K0 < OUTER) ? (np - K0) : OUTER;
      if (!trailing_update(np, K0, w, dstart, agg, &t)) break;
      if (oz_shape(t.rem, t.ncols, t.kd)) {
        const size_t sy = ozaki_ws_bytes(t.rem, t.ncols, t.kd, true);
        if (sy > b) b = sy;
      }
      if (t.full) dstart = K0 + w;
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
  size_t panel = ((size_t)2 * np * NB * sizeof(double) + 255) & ~size_t(255);
  const size_t tri = t_region_bytes(np);
  if (tri > panel) panel = tri;
  return HDR_BYTES + panel + oz_region_bytes(np, true);
}

namespace {
size_t p_region_bytes(int np) {
  size_t panel = ((size_t)2 * np * NB * sizeof(double) + 255) & ~size_t(255);
  const size_t tri = t_region_bytes(np);
  return tri > panel ? tri : panel;
}

// The factorisation's own streams for one call: `crit` (highest priority: leaf -> panel -> next
// block column, the dependent chain) and `side` (lowest priority: the rest of each panel's update
// inside the outer block, overlapped with the next leaf and panel).  Joined back into the
// caller's stream at the end; destroyed on every exit path (the driver frees them after the
// queued work completes).
struct PotrfStreams {
  cudaStream_t caller = nullptr, crit = nullptr, side = nullptr;
  cudaEvent_t ea = nullptr, eb = nullptr, join = nullptr;
  bool own = false;
  int open(cudaStream_t s, bool lookahead) {
    caller = crit = s;
    if (!lookahead) return GG_OK;
    int least = 0, greatest = 0;
    GG_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    GG_CUDA_TRY(cudaStreamCreateWithPriority(&crit, cudaStreamNonBlocking, greatest));
    own = true;
    GG_CUDA_TRY(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, least));
    for (cudaEvent_t* e : {&ea, &eb, &join})
      GG_CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    GG_CUDA_TRY(cudaEventRecord(join, caller));
    GG_CUDA_TRY(cudaStreamWaitEvent(crit, join, 0));
    return GG_OK;
  }
  bool closed = false;
  int close() {   // caller waits for crit (which has waited for side)
    if (!own || closed) return GG_OK;
    closed = true;
    GG_CUDA_TRY(cudaEventRecord(eb, side));
    GG_CUDA_TRY(cudaStreamWaitEvent(crit, eb, 0));
    GG_CUDA_TRY(cudaEventRecord(join, crit));
    GG_CUDA_TRY(cudaStreamWaitEvent(caller, join, 0));
    return GG_OK;
  }
  ~PotrfStreams() {
    if (!own) return;
    // an early (error) return still orders the caller's stream after every queued kernel, so the
    // caller may free the workspace as soon as its own stream says so
    if (!closed && side != nullptr && crit != nullptr) close();
    if (crit != caller && crit != nullptr) cudaStreamDestroy(crit);
    if (side != nullptr) cudaStreamDestroy(side);
    for (cudaEvent_t e : {ea, eb, join})
      if (e != nullptr) cudaEventDestroy(e);
  }
};
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
  const char* la = getenv("GG_POTRF_LOOKAHEAD");   // tuning knob: 0 = one stream, no look-ahead
  PotrfStreams st;
  GG_TRY(st.open(s, la == nullptr || la[0] != '0'));
  cudaStream_t cs_ = st.crit;
  // optional phase timing (GG_POTRF_TIMING=1): factor / inverse, to stderr (events on the
  // critical stream, no synchronisation inside the phases)
  const bool timing = getenv("GG_POTRF_TIMING") != nullptr;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  if (timing) {
    for (auto& e : ev) cudaEventCreate(&e);
    cudaEventRecord(ev[0], cs_);
  }
  // Two-level right-looking blocking: outer block columns of OUTER (= 8 leaves); inside one,
  // leaf + panel + an update restricted to the outer block's columns; after it, one trailing
  // SYRK of depth OUTER (8x the arithmetic intensity of a depth-128 update; 1024 measured best
  // between 256 and 4096 at n = 1e4 and 4e4) -- aggregated over syrk_agg() outer blocks for the
  // columns beyond the next outer block (see trailing_update).
  // Look-ahead inside the outer block: panel k's update is split into (a) the next block column
  // k+1 on the critical stream, then leaf k+1 and panel k+1 follow at once, while (b) the columns
  // beyond k+1 are updated on the side stream; the critical stream waits for (b) before its next
  // (a) (both write block column k+2).  Panels alternate between two buffers (b reads panel k
  // while panel k+1 is formed).
  const int agg = syrk_agg();
  int dstart = 0;   // first panel column whose update of the far columns is still deferred
  for (int K0 = 0; K0 < np; K0 += OUTER) {
    const int w = (np - K0 < OUTER) ? (np - K0) : OUTER;
    bool pend = false;   // side-stream update not yet waited for
    for (int k = K0; k < K0 + w; k += NB) {
      leaf_kernel<true><<<1, LEAF_THREADS, LEAF_SMEM, cs_>>>(L, ldp, Linv, ldp, k, &hdr->info);
      GG_LAUNCH_CHECK("potrf leaf_kernel");
      const int rem = np - k - NB;          // rows below this leaf
      if (rem <= 0) break;
      const int rem_in = K0 + w - k - NB;   // columns of the outer block right of this leaf
      double* Pk = P + (size_t)((k / NB) & 1) * np * NB;
      // P = A21 Dinv^T (all rows below), written back into L's column block
      GemmArgs pan{};
      pan.M = rem; pan.N = NB; pan.K = NB;
      pan.A = L + (k + NB) + (long long)k * ldp; pan.lda = ldp;
      pan.B = Linv + k + (long long)k * ldp; pan.ldb = ldp;
      pan.C = Pk; pan.ldc = np;
      pan.alpha = 1.0; pan.beta = 0.0; pan.flags = 0; pan.abort_flag = &hdr->info;
      GG_TRY(launch_dgemm(pan, true, cs_));
      GG_CUDA_TRY(cudaMemcpy2DAsync(L + (k + NB) + (long long)k * ldp,
                                    (size_t)ldp * sizeof(double), Pk, (size_t)np * sizeof(double),
                                    (size_t)rem * sizeof(double), NB, cudaMemcpyDeviceToDevice, cs_));
      if (rem_in <= 0) continue;
      if (pend) {
        GG_CUDA_TRY(cudaStreamWaitEvent(cs_, st.eb, 0));
        pend = false;
      }
      // (a) A[k+NB:, k+NB:k+2NB] -= P P[:NB]^T   (with no side stream: all rem_in columns)
      const int na = st.side ? (rem_in < NB ? rem_in : NB) : rem_in;
      GemmArgs upd{};
      upd.M = rem; upd.N = na; upd.K = NB;
      upd.A = Pk; upd.lda = np;
      upd.B = Pk; upd.ldb = np;
      upd.C = L + (k + NB) + (long long)(k + NB) * ldp; upd.ldc = ldp;
      upd.alpha = -1.0; upd.beta = 1.0; upd.flags = GEMM_C_LOWER; upd.abort_flag = &hdr->info;
      GG_TRY(launch_dgemm(upd, true, cs_));
      if (rem_in > na) {
        // (b) A[k+2NB:, k+2NB:K0+w] -= P[NB:] P[NB:rem_in]^T on the side stream
        GG_CUDA_TRY(cudaEventRecord(st.ea, cs_));
        GG_CUDA_TRY(cudaStreamWaitEvent(st.side, st.ea, 0));
        GemmArgs ub{};
        ub.M = rem - NB; ub.N = rem_in - NB; ub.K = NB;
        ub.A = Pk + NB; ub.lda = np;
        ub.B = Pk + NB; ub.ldb = np;
        ub.C = L + (k + 2 * NB) + (long long)(k + 2 * NB) * ldp; ub.ldc = ldp;
        ub.alpha = -1.0; ub.beta = 1.0; ub.flags = GEMM_C_LOWER; ub.abort_flag = &hdr->info;
        GG_TRY(launch_dgemm(ub, true, st.side));
        GG_CUDA_TRY(cudaEventRecord(st.eb, st.side));
        pend = true;
      }
    }
    if (pend) GG_CUDA_TRY(cudaStreamWaitEvent(cs_, st.eb, 0));
    TrailingUpdate t;
    if (!trailing_update(np, K0, w, dstart, agg, &t)) break;
    // trailing SYRK: A[K0+w:, K0+w : K0+w+ncols] -= Ld Ld[:ncols]^T, Ld = L[K0+w:, dstart:K0+w]
    // (the deferred panels, read in place; disjoint from the updated region), lower tiles only
    const double* Ld = L + (K0 + w) + (long long)dstart * ldp;
    double* C = L + (K0 + w) + (long long)(K0 + w) * ldp;
    if (oz != nullptr && oz_shape(t.rem, t.ncols, t.kd)) {
      GG_TRY(ozaki_gemm_run(t.rem, t.ncols, t.kd, Ld, 1, ldp, nullptr, 0, 0, C, ldp, -1.0, 1.0,
                            GEMM_C_LOWER, oz, oz_bytes, &hdr->info, cs_));
    } else {
      GemmArgs upd{};
      upd.M = t.rem; upd.N = t.ncols; upd.K = t.kd;
      upd.A = Ld; upd.lda = ldp;
      upd.B = Ld; upd.ldb = ldp;
      upd.C = C; upd.ldc = ldp;
      upd.alpha = -1.0; upd.beta = 1.0; upd.flags = GEMM_C_LOWER; upd.abort_flag = &hdr->info;
      GG_TRY(launch_dgemm(upd, true, cs_));
    }
    if (t.full) dstart = K0 + w;
  }
  if (timing) cudaEventRecord(ev[1], cs_);
  GG_TRY(trtri_offdiag(np, L, Linv, ldp, P, oz, oz_bytes, &hdr->info, cs_));
  GG_TRY(st.close());
  if (timing) {
    cudaEventRecord(ev[2], cs_);
    cudaEventSynchronize(ev[2]);
    float f = 0.f, iv = 0.f;
    cudaEventElapsedTime(&f, ev[0], ev[1]);
    cudaEventElapsedTime(&iv, ev[1], ev[2]);
    fprintf(stderr, "[gg potrf n=%d] factor %.2f ms, inverse %.2f ms\n", n, f, iv);
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
  const size_t oz_bytes = use_ozaki() ? oz_region_bytes(np, false) : 0;
  void* oz = oz_bytes ? static_cast<char*>(work) + HDR_BYTES + t_region_bytes(np) : nullptr;
  return trtri_offdiag(np, L, Linv, ldp, T, oz, oz_bytes, nullptr, s);
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

#ifdef GG_LEAF_PROFILE
extern "C" int gg_leaf_profile_read(long long* out, int n) {
  return cudaMemcpyFromSymbol(out, gg::g_leaf_ts, sizeof(long long) * (n < 64 ? n : 64)) ==
                 cudaSuccess ? 0 : 3;
}
#endif
