// FP64 GEMM on the sm_100a double-precision tensor path (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).
//
// tcgen05.mma has no f64 kind (ptxas rejects .kind::f64), so FP64 tensor work on B200 is issued
// as warp-level DMMA.  Measured on this pool's B200: DMMA 37.1 TFLOP/s sustained at 1965 MHz
// (profiles/r01_fp64_peak.log), DFMA 34 TFLOP/s, cuBLAS DGEMM 35.5 TFLOP/s.
//
// This one kernel is the workhorse of the hot path:
//   * the streamed TRSM  Xbar = Linv * X       (A lower-triangular, heavy row tiles first)
//   * the Cholesky panel L21 = A21 * Dinv^T    (op(B) = B^T)
//   * the Cholesky trailing update A22 -= P P^T (lower tiles only)
//   * the recursive triangular inverse          (triangular A or B)
// Tile: 128 x 128 x 16, 8 warps (2 x 4), warp tile 64 x 32 = 8 x 4 DMMA fragments, 4-stage
// cp.async pipeline (149 KB smem, 1 CTA / SM).  Every output element is accumulated in the
// same k order regardless of its tile position, so per-column results are bitwise independent
// of the column's position in the block (tests/test_kernel.py:228-241 in the reference).
#include <cstdlib>

#include "gg_internal.cuh"

namespace gg {
namespace {

// Tile shapes: the big tile (128 x 128, 8 warps of 64 x 32) and, for problems that do not fill
// the GPU with big tiles (the factorisation's panel and next-column updates: a 128-column strip
// of up to ~300 row tiles, on the critical path), a small one (64 x 64, 4 warps of 32 x 32:
// 4x the CTAs, up to 6 resident per SM).
struct BigTile { static constexpr int BM = 128, BN = 128, WM = 2, WN = 4, FM = 8, FN = 4; };
struct SmallTile { static constexpr int BM = 64, BN = 64, WM = 2, WN = 2, FM = 4, FN = 4; };
constexpr int BK = 16, STAGES = 4;

template <class T> constexpr int nthreads() { return T::WM * T::WN * 32; }
template <class T> constexpr int as_ld() { return T::BM + 4; }   // As[k][m], +4: conflict-free
template <class T, bool BT> constexpr int bs_ld() { return BT ? T::BN + 4 : BK + 4; }
template <class T> constexpr int a_stage() { return BK * as_ld<T>(); }
template <class T, bool BT> constexpr int b_stage() { return BT ? BK * bs_ld<T, BT>() : T::BN * bs_ld<T, BT>(); }
template <class T, bool BT>
constexpr size_t smem_bytes() { return size_t(STAGES) * (a_stage<T>() + b_stage<T, BT>()) * sizeof(double); }

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 16 : 0;   // src-size 0 -> zero fill (out-of-range columns)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// D = A(8x4) * B(4x8) + D.  Lane (g = lane>>2, t = lane&3) holds A[g][t], B[t][g],
// D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <class T, bool BT>
__global__ void __launch_bounds__(nthreads<T>()) dgemm_dmma_kernel(GemmArgs a) {
  constexpr int BM = T::BM, BN = T::BN, NT = nthreads<T>();
  constexpr int FM = T::FM, FN = T::FN;            // DMMA fragments per warp (rows, columns)
  constexpr int AS_LD = as_ld<T>(), BS_LD = bs_ld<T, BT>();
  constexpr int A_STAGE = a_stage<T>(), B_STAGE = b_stage<T, BT>();
  if (a.abort_flag != nullptr && *a.abort_flag != 0) return;
  if (blockIdx.y) {   // strided batch
    a.A += blockIdx.y * a.sA;
    a.B += blockIdx.y * a.sB;
    a.C += blockIdx.y * a.sC;
  }
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;

  const int num_mt = a.M / BM;
  const int num_nt = (a.N + BN - 1) / BN;
  const int bid = blockIdx.x;
  int mt, nt;
  if (a.flags & GEMM_A_LOWER) {
    // triangular A: the last row tiles carry the longest k range -> schedule them first;
    // consecutive CTAs share the same A row panel (L2 reuse of Linv).
    mt = num_mt - 1 - bid / num_nt;
    nt = bid % num_nt;
  } else {
    mt = bid % num_mt;
    nt = bid / num_mt;
  }
  const int m0 = mt * BM, n0 = nt * BN;
  if ((a.flags & GEMM_C_LOWER) && n0 >= m0 + BM) return;   // strictly above the diagonal
  int k_begin = 0, k_end = a.K;
  if (a.flags & GEMM_A_LOWER) k_end = min(a.K, m0 + BM);
  if (a.flags & GEMM_B_LOWER) k_begin = min(a.K, n0);
  const int nk = (k_end > k_begin) ? (k_end - k_begin) / BK : 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / T::WN, wn = warp % T::WN;

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = k_begin + kt * BK;
    double* as = As + stage * A_STAGE;
    double* bs = Bs + stage * B_STAGE;
#pragma unroll
    for (int c = tid; c < BK * BM / 2; c += NT) {   // 16-byte chunks of A (m contiguous)
      const int kc = c / (BM / 2), mc = c % (BM / 2);
      cp_async16(as + kc * AS_LD + mc * 2, a.A + (long long)(k0 + kc) * a.lda + m0 + mc * 2, true);
    }
    if (BT) {
#pragma unroll
      for (int c = tid; c < BK * BN / 2; c += NT) {
        const int kr = c / (BN / 2), nc = c % (BN / 2);
        const int col = n0 + nc * 2;
        const bool pred = col < a.N;
        const double* src = a.B + (long long)(k0 + kr) * a.ldb + (pred ? col : 0);
        cp_async16(bs + kr * BS_LD + nc * 2, src, pred);
      }
    } else {
#pragma unroll
      for (int c = tid; c < BN * BK / 2; c += NT) {
        const int nc = c / (BK / 2), kch = c % (BK / 2);
        const int col = n0 + nc;
        const bool pred = col < a.N;
        const double* src = a.B + (long long)(pred ? col : 0) * a.ldb + k0 + kch * 2;
        cp_async16(bs + nc * BS_LD + kch * 2, src, pred);
      }
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int pf = kt + STAGES - 1;
    if (pf < nk) load_stage(pf % STAGES, pf);
    cp_async_commit();

    const double* as = As + (kt % STAGES) * A_STAGE + wm * (8 * FM) + g;
    const double* bs = Bs + (kt % STAGES) * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = as[(kk + t) * AS_LD + i * 8];
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        bf[j] = BT ? bs[(kk + t) * BS_LD + wn * (8 * FN) + j * 8 + g]
                   : bs[(wn * (8 * FN) + j * 8 + g) * BS_LD + kk + t];
      }
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  const double alpha = a.alpha, beta = a.beta;
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int row = m0 + wm * (8 * FM) + i * 8 + g;
#pragma unroll
    for (int j = 0; j < FN; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn * (8 * FN) + j * 8 + 2 * t + e;
        if (col < a.N) {
          double* cp = a.C + (long long)col * a.ldc + row;
          const double v = acc[i][j][e];
          *cp = (beta == 0.0) ? alpha * v : fma(alpha, v, beta * *cp);
        }
      }
    }
  }
}

template <class T, bool BT>
int launch_tiles(const GemmArgs& a, cudaStream_t s) {
  const long long tiles = (long long)(a.M / T::BM) * ((a.N + T::BN - 1) / T::BN);
  if (tiles > 0x7fffffffLL || a.batch > 65535) {
    set_error("dgemm: too many tiles");
    return GG_EDIM;
  }
  const dim3 grid((unsigned)tiles, a.batch > 1 ? (unsigned)a.batch : 1u);
  GG_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<T, BT>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_bytes<T, BT>()));
  dgemm_dmma_kernel<T, BT><<<grid, nthreads<T>(), smem_bytes<T, BT>(), s>>>(a);
  GG_LAUNCH_CHECK("dgemm_dmma_kernel launch");
  return GG_OK;
}

}  // namespace

int launch_dgemm(const GemmArgs& a, bool trans_b, cudaStream_t s) {
  if (a.M < 0 || a.N < 0 || a.K < 0 || a.M % BigTile::BM != 0 || a.K % BK != 0) {
    set_error("dgemm: M must be a multiple of 128 and K a multiple of 16");
    return GG_EDIM;
  }
  if (trans_b && a.N % 2 != 0) {
    set_error("dgemm: op(B)=B^T needs an even column count");
    return GG_EDIM;
  }
  if ((a.flags & GEMM_C_LOWER) && a.N > a.M) {
    set_error("dgemm: lower-only output needs N <= M (C anchored on the diagonal)");
    return GG_EDIM;
  }
  if (a.M == 0 || a.N == 0) return GG_OK;
  if (a.lda < a.M || a.ldc < a.M || a.ldb < (trans_b ? a.N : a.K)) {
    set_error("dgemm: leading dimension too small");
    return GG_EDIM;
  }
  // fewer big tiles than SMs (x batch): the small tile keeps the GPU busy
  const long long big = (long long)(a.M / BigTile::BM) * ((a.N + BigTile::BN - 1) / BigTile::BN) *
                        (a.batch > 1 ? a.batch : 1);
  // short k (the factorisation's K = 128 updates: 8 k-steps per big tile, one CTA per SM, nothing
  // to hide a tile's prologue / C read-modify-write behind) -> small tiles too, several per SM
  static const int kmax_small = [] {
    const char* v = getenv("GG_DGEMM_SMALL_K");   // tuning knob (0: only the sub-wave rule)
    return v ? atoi(v) : 128;   // measured r02: 128 best (n = 4e4 prepare -3%, 256 worse)
  }();
  const bool small = (big < 148 || a.K <= kmax_small) && !(trans_b && a.N % 2 != 0);
  if (small) return trans_b ? launch_tiles<SmallTile, true>(a, s) : launch_tiles<SmallTile, false>(a, s);
  return trans_b ? launch_tiles<BigTile, true>(a, s) : launch_tiles<BigTile, false>(a, s);
}

}  // namespace gg
