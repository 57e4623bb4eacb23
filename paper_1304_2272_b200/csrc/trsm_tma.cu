// Streamed TRSM  Xbar = Linv * X  as a persistent, warp-specialised TMA + DMMA kernel (sm_100a).
//
// The dominant cost of the GLS sweep (n^2 FLOP per SNP).  Design:
//   * operands are K-major: A = Linv stored row-major ("LinvT", k contiguous per row m, upper part
//     zero) and B = X column-major (k contiguous per SNP column); both are moved by TMA
//     (cp.async.bulk.tensor.2d) as 128 x 16 FP64 boxes with the 128-byte swizzle;
//   * warp 8 is the producer: one elected lane walks the CTA's tile sequence and keeps a
//     6-stage ring of (A, B) boxes full (mbarrier full/empty pairs, expect_tx byte counts);
//   * warps 0-7 are consumers: 2 x 4 warp grid, 64 x 32 warp tile = 8 x 4 DMMA.8x8x4 fragments;
//     no CTA-wide barrier in the main loop — a warp waits only on the stage it needs;
//   * fragment rows/columns are permuted (row = 16*(i/2) + 2*g + (i&1)) so the swizzled
//     fragment loads are bank-conflict free and the two row-fragments of a pair store as one
//     16-byte vector per lane (4 full 128-byte lines per warp store);
//   * persistent grid (one CTA per SM), tiles in heavy-first order dealt in a snake so the
//     triangular work (row tile mt needs k < (mt+1)*128) balances across SMs; the producer runs
//     ahead across tile boundaries, hiding each tile's prologue behind the previous epilogue.
// Per-element accumulation order (k ascending in DMMA k=4 chunks) is the same as the cp.async
// GEMM (gemm_f64.cu), so both kernels give bitwise-identical Xbar columns.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <string>

#include "gg_internal.cuh"

namespace gg {
namespace {

constexpr int BM = 128, BN = 128, BK = 16;
constexpr int STAGES = 6;
constexpr int CONSUMER_WARPS = 8;
constexpr int THREADS = (CONSUMER_WARPS + 1) * 32;
constexpr int TILE_BYTES = BM * BK * 8;                 // 16 KB per operand box
constexpr int STAGE_BYTES = 2 * TILE_BYTES;
constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct TrsmArgs {
  int N;          // columns (SNPs)
  int num_mt;     // np / 128
  int num_nt;     // ceil(N / 128)
  double* C;
  long long ldc;
  const int* gate;   // run only if *gate == gate_value (nullptr: always)
  int gate_value;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, unsigned bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* map, unsigned bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// tile t of the heavy-first order -> (mt, nt)
__device__ __forceinline__ void tile_coords(int t, int num_mt, int num_nt, int& mt, int& nt) {
  mt = num_mt - 1 - t / num_nt;
  nt = t % num_nt;
}

// r-th tile handled by CTA b of G (snake deal)
__device__ __forceinline__ int tile_of(int r, int b, int G) {
  return r * G + ((r & 1) ? (G - 1 - b) : b);
}

// PACKED = false: A is the full row-major inverse (2D map, box at (k, m)).
// PACKED = true : A is the packed tile-major lower inverse (3D map over 128 x 16 tiles, tile index
//                 4*mt*(mt+1) + kt; only the tiles on or below the diagonal exist).
template <bool PACKED>
__global__ void __launch_bounds__(THREADS, 1)
    trsm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    TrsmArgs a) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + STAGES * STAGE_BYTES);
  const unsigned sbase = smem_u32(smem);
  const unsigned full0 = smem_u32(bars);
  const unsigned empty0 = smem_u32(bars + STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (a.gate != nullptr && *a.gate != a.gate_value) return;   // device-side path selection
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, CONSUMER_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int total = a.num_mt * a.num_nt;
  const int G = gridDim.x, b = blockIdx.x;

  if (warp == CONSUMER_WARPS) {
    // ------------------------------ producer -------------------------------------------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<unsigned long long>(&tmA))
                   : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<unsigned long long>(&tmB))
                   : "memory");
      int stage = 0;
      unsigned phase = 0;
      for (int r = 0;; ++r) {
        const int t = tile_of(r, b, G);
        if (t >= total) break;
        int mt, nt;
        tile_coords(t, a.num_mt, a.num_nt, mt, nt);
        const int nk = (mt + 1) * (BM / BK);   // triangular: k < (mt+1)*128
        for (int kt = 0; kt < nk; ++kt) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const unsigned fb = full0 + 8 * stage;
          mbar_expect_tx(fb, STAGE_BYTES);
          const unsigned dA = sbase + stage * STAGE_BYTES;
          if (PACKED) tma_load_3d(dA, &tmA, fb, 0, 0, 4 * mt * (mt + 1) + kt);
          else tma_load_2d(dA, &tmA, fb, kt * BK, mt * BM);
          tma_load_2d(dA + TILE_BYTES, &tmB, fb, kt * BK, nt * BN);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // -------------------------------- consumers ------------------------------------------------
  const int g = lane >> 2, tq = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  // byte offsets of this lane's fragment rows inside a 128-row swizzled box, and their swizzle
  unsigned a_row[8], b_row[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a_row[i] = (wm * 64 + 16 * (i >> 1) + 2 * g + (i & 1));
#pragma unroll
  for (int j = 0; j < 4; ++j) b_row[j] = (wn * 32 + 16 * (j >> 1) + 2 * g + (j & 1));

  int stage = 0;
  unsigned phase = 0;
  for (int r = 0;; ++r) {
    const int t = tile_of(r, b, G);
    if (t >= total) break;
    int mt, nt;
    tile_coords(t, a.num_mt, a.num_nt, mt, nt);
    const int nk = (mt + 1) * (BM / BK);
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < nk; ++kt) {
      mbar_wait(full0 + 8 * stage, phase);
      const unsigned char* As = smem + stage * STAGE_BYTES;
      const unsigned char* Bs = As + TILE_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        const unsigned kc = (unsigned)((kk >> 1) | (tq >> 1));   // 16-byte chunk of k = kk + tq
        const unsigned ks = (unsigned)(tq & 1) << 3;
        double af[8], bf[4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          af[i] = *reinterpret_cast<const double*>(As + a_row[i] * 128 +
                                                   ((kc ^ (a_row[i] & 7)) << 4) + ks);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          bf[j] = *reinterpret_cast<const double*>(Bs + b_row[j] * 128 +
                                                   ((kc ^ (b_row[j] & 7)) << 4) + ks);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * stage);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }

    // epilogue: rows (2g, 2g+1) of a fragment pair are adjacent -> one 16-byte store
    const long long m_base = (long long)mt * BM + wm * 64 + 2 * g;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = nt * BN + wn * 32 + 16 * (j >> 1) + 4 * tq + 2 * e + (j & 1);
        if (col < a.N) {
          double* cp = a.C + (long long)col * a.ldc + m_base;
#pragma unroll
          for (int ip = 0; ip < 4; ++ip) {
            double2 v = make_double2(acc[2 * ip][j][e], acc[2 * ip + 1][j][e]);
            *reinterpret_cast<double2*>(cp + 16 * ip) = v;
          }
        }
      }
    }
  }
}

// ---- skinny right-hand sides (the prepare's [X_L | y]: nrhs <= 16) ------------------------------
// The tiled kernel above computes 128 columns per tile, so for a handful of covariate columns it
// spends its DMMA time on padding and its grid on 79 row tiles (1.39 ms at n = 1e4).  Here a CTA
// owns 32 rows x up to 16 columns and streams its slice of the packed inverse (4 KB per 16-k
// tile, contiguous) through a cp.async ring, bandwidth-bound; heavy row blocks first.  Each
// element is accumulated by the same DMMA.8x8x4 sequence as the tiled kernel (k ascending from 0
// in chunks of 4, accumulator from zero), so a column's X-bar is bitwise the same whichever
// kernel whitens it (tests/test_gpu_kernel.py::test_skinny_trsm_bitwise_equal_to_tiled).
constexpr int SK_ROWS = 32, SK_COLS = 16, SK_STAGES = 6, SK_THREADS = 128;
constexpr int SK_LD = BK + 4;   // smem row stride (doubles): conflict-free DMMA fragment reads
constexpr int SK_A = SK_ROWS * SK_LD, SK_B = SK_COLS * SK_LD;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(pred ? 16 : 0)
               : "memory");
}

__global__ void __launch_bounds__(SK_THREADS) trsm_skinny_kernel(
    int num_rb, int nrhs, const double* __restrict__ LinvP, const double* __restrict__ B,
    long long ldb, double* __restrict__ X, long long ldx, const int* gate, int gate_value) {
  if (gate != nullptr && *gate != gate_value) return;   // device-side path selection
  __shared__ __align__(16) double As[SK_STAGES][SK_A];
  __shared__ __align__(16) double Bs[SK_STAGES][SK_B];
  const int rb = num_rb - 1 - blockIdx.x;                 // heavy (long k range) first
  const int mt = rb >> 2, sub = rb & 3;
  const int nk = (mt + 1) * (BM / BK);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* Abase = LinvP + (long long)4 * mt * (mt + 1) * (BM * BK) + sub * SK_ROWS * BK;
  auto load = [&](int st, int kt) {
    const double* a = Abase + (long long)kt * (BM * BK);
#pragma unroll
    for (int c = tid; c < SK_ROWS * (BK / 2); c += SK_THREADS) {   // 2 doubles per chunk
      const int r = c / (BK / 2), q = c % (BK / 2);
      cp_async16(&As[st][r * SK_LD + 2 * q], a + r * BK + 2 * q, true);
    }
    {
      const int j = tid / (BK / 2), q = tid % (BK / 2);
      const bool ok = j < nrhs;
      cp_async16(&Bs[st][j * SK_LD + 2 * q], B + (ok ? (long long)j * ldb : 0) + kt * BK + 2 * q, ok);
    }
  };
#pragma unroll
  for (int st = 0; st < SK_STAGES - 1; ++st) {
    if (st < nk) load(st, st);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  const int g = lane >> 2, t = lane & 3;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(SK_STAGES - 2) : "memory");
    __syncthreads();
    const int pf = kt + SK_STAGES - 1;
    if (pf < nk) load(pf % SK_STAGES, pf);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const double* a = As[kt % SK_STAGES] + (8 * warp + g) * SK_LD + t;
    const double* b = Bs[kt % SK_STAGES] + g * SK_LD + t;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const double af = a[kk];
      dmma(acc[0], af, b[kk]);
      dmma(acc[1], af, b[8 * SK_LD + kk]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  const long long row = (long long)rb * SK_ROWS + 8 * warp + g;
#pragma unroll
  for (int nf = 0; nf < 2; ++nf)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int col = 8 * nf + 2 * t + e;
      if (col < nrhs) X[row + (long long)col * ldx] = acc[nf][e];
    }
}

// ---- tensor maps ----------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// K-major FP64 operand: `rows` rows of `kdim` contiguous doubles, row stride ld (doubles).
int make_kmajor_map(CUtensorMap* map, const double* base, long long kdim, long long rows,
                    long long ld) {
  auto fn = encode_fn();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return GG_ECUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {BK, BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
    return GG_ECUDA;
  }
  return GG_OK;
}

__global__ void transpose_kernel(int np, const double* __restrict__ A, long long lda,
                                 double* __restrict__ T, long long ldt) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y)
    tile[j][threadIdx.x] = A[(long long)(bx + j) * lda + by + threadIdx.x];   // column bx+j
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y)
    T[(long long)(by + j) * ldt + bx + threadIdx.x] = tile[threadIdx.x][j];
}

// col-major (or row-major) lower inverse -> packed tile-major 128 x 16 tiles (k contiguous)
__global__ void pack_lower_kernel(int np, const double* __restrict__ A, long long ld, int row_major,
                                  double* __restrict__ P) {
  const int nmt = np / BM;
  const long long ntile = 4LL * nmt * (nmt + 1);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ntile * 2048;
       e += (long long)gridDim.x * blockDim.x) {
    const long long t = e >> 11;
    const int within = (int)(e & 2047), r = within >> 4, kk = within & 15;
    // invert t = 4*mt*(mt+1) + kt with 0 <= kt < 8*(mt+1)
    int mt = (int)((sqrt(1.0 + (double)t) - 1.0) / 2.0);
    while (4LL * (mt + 1) * (mt + 2) <= t) ++mt;
    while (4LL * mt * (mt + 1) > t) --mt;
    const int kt = (int)(t - 4LL * mt * (mt + 1));
    const long long i = (long long)mt * BM + r, k = (long long)kt * BK + kk;
    const double v = (k <= i) ? (row_major ? A[k + i * ld] : A[i + k * ld]) : 0.0;
    P[e] = v;
  }
}

// The same packed layout assembled from one rank's share of a 2D block-cyclic inverse (block nb,
// grid gr x gc, this rank at (pr, pc), local column-major with leading dimension ldl).  Tiles the
// rank does not own are written as zeros, so summing every rank's buffer (an all-reduce over
// disjoint supports) reproduces the full packed inverse exactly.
__global__ void pack_lower_bc_kernel(int np, int nb, int gr, int gc, int pr, int pc,
                                     const double* __restrict__ B, long long ldl,
                                     double* __restrict__ P) {
  const int nmt = np / BM;
  const long long ntile = 4LL * nmt * (nmt + 1);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ntile * 2048;
       e += (long long)gridDim.x * blockDim.x) {
    const long long t = e >> 11;
    const int within = (int)(e & 2047), r = within >> 4, kk = within & 15;
    int mt = (int)((sqrt(1.0 + (double)t) - 1.0) / 2.0);
    while (4LL * (mt + 1) * (mt + 2) <= t) ++mt;
    while (4LL * mt * (mt + 1) > t) --mt;
    const int kt = (int)(t - 4LL * mt * (mt + 1));
    const long long i = (long long)mt * BM + r, k = (long long)kt * BK + kk;
    double v = 0.0;
    if (k <= i) {
      const long long I = i / nb, J = k / nb;
      if (I % gr == pr && J % gc == pc) {
        const long long li = (I / gr) * nb + i % nb, lk = (J / gc) * nb + k % nb;
        v = B[li + lk * ldl];
      }
    }
    P[e] = v;
  }
}

int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

int transpose_square_run(int np, const double* A, int lda, double* T, int ldt, cudaStream_t s) {
  if (np % 32 != 0 || lda < np || ldt < np) {
    set_error("transpose: np must be a multiple of 32 and ld >= np");
    return GG_EDIM;
  }
  dim3 grid(np / 32, np / 32), block(32, 8);
  transpose_kernel<<<grid, block, 0, s>>>(np, A, lda, T, ldt);
  GG_LAUNCH_CHECK("transpose_kernel");
  return GG_OK;
}

size_t packed_lower_elems(int n) {
  const long long nmt = pad_rows(n) / BM;
  return (size_t)(4LL * nmt * (nmt + 1)) * 2048;
}

int pack_lower_run(int n, const double* A, int lda, int row_major, double* P, cudaStream_t s) {
  const int np = pad_rows(n);
  if (lda < np) {
    set_error("pack_lower: lda must be >= gg_pad(n)");
    return GG_EDIM;
  }
  long long grid = ((long long)packed_lower_elems(n) + 255) / 256;
  if (grid > 148LL * 64) grid = 148LL * 64;
  pack_lower_kernel<<<(int)grid, 256, 0, s>>>(np, A, lda, row_major, P);
  GG_LAUNCH_CHECK("pack_lower_kernel");
  return GG_OK;
}

int pack_lower_bc_run(int n, int nb, int gr, int gc, int pr, int pc, const double* B, int ldl,
                      double* P, cudaStream_t s) {
  if (nb < BM || nb % BM != 0 || gr < 1 || gc < 1 || pr < 0 || pr >= gr || pc < 0 || pc >= gc) {
    set_error("pack_lower_blockcyclic: nb must be a multiple of 128 and (pr, pc) inside the grid");
    return GG_EARG;
  }
  long long grid = ((long long)packed_lower_elems(n) + 255) / 256;
  if (grid > 148LL * 64) grid = 148LL * 64;
  pack_lower_bc_kernel<<<(int)grid, 256, 0, s>>>(pad_rows(n), nb, gr, gc, pr, pc, B, ldl, P);
  GG_LAUNCH_CHECK("pack_lower_bc_kernel");
  return GG_OK;
}

static int make_packed_map(CUtensorMap* map, const double* base, long long ntiles) {
  auto fn = encode_fn();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return GG_ECUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)BK, (cuuint64_t)BM, (cuuint64_t)ntiles};
  cuuint64_t strides[2] = {(cuuint64_t)BK * sizeof(double), (cuuint64_t)BK * BM * sizeof(double)};
  cuuint32_t box[3] = {BK, BM, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (packed) failed (code " + std::to_string((int)r) + ")");
    return GG_ECUDA;
  }
  return GG_OK;
}

template <bool PACKED>
static int launch_trsm(const CUtensorMap& mA, const CUtensorMap& mB, int np, int nrhs, double* X,
                       int ldx, cudaStream_t s, const int* gate = nullptr, int gate_value = 0) {
  TrsmArgs a;
  a.gate = gate;
  a.gate_value = gate_value;
  a.N = nrhs;
  a.num_mt = np / BM;
  a.num_nt = (nrhs + BN - 1) / BN;
  a.C = X;
  a.ldc = ldx;
  const int tiles = a.num_mt * a.num_nt;
  int grid = sm_count();
  if (grid > tiles) grid = tiles;
  GG_CUDA_TRY(cudaFuncSetAttribute(trsm_tma_kernel<PACKED>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
  trsm_tma_kernel<PACKED><<<grid, THREADS, SMEM_BYTES, s>>>(mA, mB, a);
  GG_LAUNCH_CHECK("trsm_tma_kernel");
  return GG_OK;
}

int trsm_packed_run(int n, int nrhs, const double* LinvP, const double* B, int ldb, double* X,
                    int ldx, cudaStream_t s) {
  return trsm_packed_gated_run(n, nrhs, LinvP, B, ldb, X, ldx, nullptr, 0, s);
}

int trsm_packed_gated_run(int n, int nrhs, const double* LinvP, const double* B, int ldb,
                          double* X, int ldx, const int* gate, int gate_value, cudaStream_t s) {
  const int np = pad_rows(n);
  if (ldb < np || ldx < np) {
    set_error("trsm: leading dimensions must be >= gg_pad(n)");
    return GG_EDIM;
  }
  if (nrhs <= 0) return GG_OK;
  if ((reinterpret_cast<uintptr_t>(LinvP) | reinterpret_cast<uintptr_t>(B) |
       reinterpret_cast<uintptr_t>(X)) & 15) {
    set_error("trsm: operands must be 16-byte aligned");
    return GG_EARG;
  }
  if (nrhs <= SK_COLS && (ldb & 1) == 0) {   // skinny right-hand sides (16-byte aligned columns)
    trsm_skinny_kernel<<<np / SK_ROWS, SK_THREADS, 0, s>>>(np / SK_ROWS, nrhs, LinvP, B, ldb, X,
                                                            ldx, gate, gate_value);
    GG_LAUNCH_CHECK("trsm_skinny_kernel");
    return GG_OK;
  }
  CUtensorMap mA, mB;
  const long long nmt = np / BM;
  int rc = make_packed_map(&mA, LinvP, 4LL * nmt * (nmt + 1));
  if (rc != GG_OK) return rc;
  rc = make_kmajor_map(&mB, B, np, nrhs, ldb);
  if (rc != GG_OK) return rc;
  return launch_trsm<true>(mA, mB, np, nrhs, X, ldx, s, gate, gate_value);
}

int trsm_rowmajor_run(int n, int nrhs, const double* LinvT, int ldp, const double* B, int ldb,
                      double* X, int ldx, cudaStream_t s) {
  const int np = pad_rows(n);
  if (ldp < np || ldb < np || ldx < np) {
    set_error("trsm: leading dimensions must be >= gg_pad(n)");
    return GG_EDIM;
  }
  if (nrhs <= 0) return GG_OK;
  if ((reinterpret_cast<uintptr_t>(LinvT) | reinterpret_cast<uintptr_t>(B) |
       reinterpret_cast<uintptr_t>(X)) & 15) {
    set_error("trsm: operands must be 16-byte aligned");
    return GG_EARG;
  }
  CUtensorMap mA, mB;
  int rc = make_kmajor_map(&mA, LinvT, np, np, ldp);
  if (rc != GG_OK) return rc;
  rc = make_kmajor_map(&mB, B, np, nrhs, ldb);
  if (rc != GG_OK) return rc;
  return launch_trsm<false>(mA, mB, np, nrhs, X, ldx, s);
}

}  // namespace gg
