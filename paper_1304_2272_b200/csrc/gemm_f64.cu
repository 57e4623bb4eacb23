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
#include "gg_internal.cuh"

namespace gg {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, NTHREADS = 256;
constexpr int AS_LD = BM + 4;    // As[k][m]  (m contiguous), +4 doubles: conflict-free A fragments
constexpr int BSN_LD = BK + 4;   // Bs[n][k]  (k contiguous) for op(B) = B
constexpr int BST_LD = BN + 4;   // Bs[k][n]  (n contiguous) for op(B) = B^T
constexpr int A_STAGE = BK * AS_LD;
constexpr int B_STAGE_N = BN * BSN_LD;
constexpr int B_STAGE_T = BK * BST_LD;

template <bool BT>
__host__ __device__ constexpr int b_stage() { return BT ? B_STAGE_T : B_STAGE_N; }
template <bool BT>
constexpr size_t smem_bytes() { return size_t(STAGES) * (A_STAGE + b_stage<BT>()) * sizeof(double); }

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

template <bool BT>
__global__ void __launch_bounds__(NTHREADS, 1) dgemm_dmma_kernel(GemmArgs a) {
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
  if ((a.flags & GEMM_C_LOWER) && nt > mt) return;
  const int m0 = mt * BM, n0 = nt * BN;
  int k_begin = 0, k_end = a.K;
  if (a.flags & GEMM_A_LOWER) k_end = min(a.K, m0 + BM);
  if (a.flags & GEMM_B_LOWER) k_begin = min(a.K, n0);
  const int nk = (k_end > k_begin) ? (k_end - k_begin) / BK : 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = k_begin + kt * BK;
    double* as = As + stage * A_STAGE;
    double* bs = Bs + stage * b_stage<BT>();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int c = tid + r * NTHREADS;
      const int kc = c >> 6, mc = c & 63;
      cp_async16(as + kc * AS_LD + mc * 2, a.A + (long long)(k0 + kc) * a.lda + m0 + mc * 2, true);
    }
    if (BT) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int c = tid + r * NTHREADS;
        const int kr = c >> 6, nc = c & 63;
        const int col = n0 + nc * 2;
        const bool pred = col < a.N;
        const double* src = a.B + (long long)(k0 + kr) * a.ldb + (pred ? col : 0);
        cp_async16(bs + kr * BST_LD + nc * 2, src, pred);
      }
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int c = tid + r * NTHREADS;
        const int nc = c >> 3, kch = c & 7;
        const int col = n0 + nc;
        const bool pred = col < a.N;
        const double* src = a.B + (long long)(pred ? col : 0) * a.ldb + k0 + kch * 2;
        cp_async16(bs + nc * BSN_LD + kch * 2, src, pred);
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

    const double* as = As + (kt % STAGES) * A_STAGE + wm * 64 + g;
    const double* bs = Bs + (kt % STAGES) * b_stage<BT>();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = as[(kk + t) * AS_LD + i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bf[j] = BT ? bs[(kk + t) * BST_LD + wn * 32 + j * 8 + g]
                   : bs[(wn * 32 + j * 8 + g) * BSN_LD + kk + t];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  const double alpha = a.alpha, beta = a.beta;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = m0 + wm * 64 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn * 32 + j * 8 + 2 * t + e;
        if (col < a.N) {
          double* cp = a.C + (long long)col * a.ldc + row;
          const double v = acc[i][j][e];
          *cp = (beta == 0.0) ? alpha * v : fma(alpha, v, beta * *cp);
        }
      }
    }
  }
}

}  // namespace

int launch_dgemm(const GemmArgs& a, bool trans_b, cudaStream_t s) {
  if (a.M < 0 || a.N < 0 || a.K < 0 || a.M % BM != 0 || a.K % BK != 0) {
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
  const long long tiles = (long long)(a.M / BM) * ((a.N + BN - 1) / BN);
  if (tiles > 0x7fffffffLL || a.batch > 65535) {
    set_error("dgemm: too many tiles");
    return GG_EDIM;
  }
  const dim3 grid((unsigned)tiles, a.batch > 1 ? (unsigned)a.batch : 1u);
  if (trans_b) {
    GG_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_bytes<true>()));
    dgemm_dmma_kernel<true><<<grid, NTHREADS, smem_bytes<true>(), s>>>(a);
  } else {
    GG_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_bytes<false>()));
    dgemm_dmma_kernel<false><<<grid, NTHREADS, smem_bytes<false>(), s>>>(a);
  }
  GG_LAUNCH_CHECK("dgemm_dmma_kernel launch");
  return GG_OK;
}

}  // namespace gg
