// FP64 GEMM on the int8 tensor cores (Ozaki scheme): C = beta C + alpha A B^T for FP64 operands,
// used for the large updates of the Cholesky factorisation (potrf_f64.cu).
//
// FP64 has no tcgen05 kind on sm_100a; the DMMA path peaks at 37 TFLOP/s while the int8 tensor
// cores do 4.4 POPS.  Each row i of A (and row j of B) is split error-free into 7 int8 slices of
// balanced base-256 digits below its own power of two (|A[i,:]| < 127/256 2^e_i):
//     A[i,k] = 2^e_i sum_{s=0..6} a_s[i,k] 2^(-8 (s+1)),   a_s in [-128, 127]
// (the digits of RN(A[i,k] 2^(56 - e_i)): one rounding, then exact integer digit extraction), so
//     (A B^T)[i,j] = 2^(e_i + f_j) sum_d D_d[i,j] 2^(-8 (d+2)),   D_d = sum_{s+t=d} a_s b_t^T.
// The 28 slice products with s + t <= 6 are issued as tcgen05.mma.kind::i8 into 7 int32 TMEM
// accumulators (one per diagonal d, 64 columns each); every D_d is exact for K <= 18724
// (7 2^14 K < 2^31; the host splits K into launches of <= 8192).  The dropped terms (s+t >= 7)
// are below 2^-56 of 2^(e_i+f_j) per product term and, every digit below the top one being
// centred on zero, keep random signs and cancel along k -- measured as accurate as FP64 GEMM and
// ~2x closer to the exact product than the r02 form (8 slices of 7-bit sign-magnitude digits, 36
// products; OZ_DIGIT_BITS=7 builds it, tools/oz_accuracy.py).  The epilogue forms the exact int64
// halves hi = D_0..D_3, lo = D_4..D_6 (base 2^8) and rounds once: r = 2^E fma(hi, 2^-40, lo 2^-64);
// then C = beta C + alpha r.
//
// Kernel (persistent, one CTA per SM in clusters of 2, 10 warps): warp 0 TMA producer (per 64-k
// stage: 8 slice slots of a 128-row A tile -- half of them loaded here and multicast to the
// cluster peer, which computes the neighbouring 64 columns; the 8th slot is out of bounds of the
// 7-slice operand, zero-filled by TMA and never multiplied -- and of a 64-row B tile, 96 KB,
// SWIZZLE_64B, 2-stage ring; r02: 64-byte rows halve the L2 requests of the 32-byte-row 4-stage
// form, whose operand stream was the limiter), warp 1 MMA issuer (one lane, M = 128 x N = 64..256
// x K = 32, 2 x 10 MMAs covering the 28 slice products per stage), warps 2-9 epilogue (TMEM lane =
// tile row, two warps per lane quarter, 32 columns each; release TMEM once the tile is in
// registers, then update C).
// Operand entries outside a triangular operand's triangle are sliced as zeros.
// Results are bitwise deterministic (exact integer accumulation, fixed rounding).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <string>

#include "gg_internal.cuh"

namespace gg {
namespace {

#ifndef OZ_DIGIT_BITS
#define OZ_DIGIT_BITS 8   // r02: 28 products instead of 36, n = 4e4 prepare 0.70 -> 0.61 s
#endif
// digits: 8 slices of 7-bit sign-magnitude digits (36 products, s + t <= 7) or 7 slices of 8-bit
// balanced digits (28 products, s + t <= 6) -- both keep ~56 bits below the row maximum
constexpr int OZ_DB = OZ_DIGIT_BITS;
static_assert(OZ_DB == 7 || OZ_DB == 8, "digit width");
constexpr int OZ_S = OZ_DB == 8 ? 7 : 8;   // slices per operand (= diagonals kept)
constexpr int OZ_SS = 8;                   // slice slots per stage in shared memory: TMA boxes of
                                           // 4 slices, a 7th-slice operand's 8th slot zero-filled
                                           // (out of bounds) and never multiplied
constexpr int OZ_BM = 128;                 // tile rows (MMA M)
constexpr int OZ_BN = 64;                  // tile columns (MMA N, one accumulator per diagonal)
#ifndef OZ_KC_BYTES
#define OZ_KC_BYTES 64   // measured r02: 64-byte rows 9% faster over the n = 4e4 prepare than 32
#endif
constexpr int OZ_KC = OZ_KC_BYTES;         // k per stage: 32 (one MMA K, 32-byte swizzled rows) or
                                           // 64 (two MMA K steps, 64-byte swizzled rows)
constexpr int OZ_STAGES = OZ_KC == 32 ? 4 : 2;
static_assert(OZ_KC == 32 || OZ_KC == 64, "k per stage");
constexpr int OZ_A_BYTES = OZ_SS * OZ_BM * OZ_KC;   // 64 KB at 64-byte stages
constexpr int OZ_B_BYTES = OZ_SS * OZ_BN * OZ_KC;   // 32 KB
constexpr int OZ_STAGE_BYTES = OZ_A_BYTES + OZ_B_BYTES;
constexpr int OZ_EPI_WARPS = 8;
constexpr int OZ_THREADS = (2 + OZ_EPI_WARPS) * 32;
constexpr size_t OZ_SMEM = size_t(OZ_STAGES) * OZ_STAGE_BYTES + 1024 + 256;
constexpr int OZ_KMAX = 8192;              // k per launch: exact int32 diagonals need
                                           // 7 * 2^14 * K < 2^31 (8 * 127^2 * K with 7-bit digits);
                                           // 8192 bounds the slice workspace
constexpr unsigned OZ_IDESC_BASE = (2u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(OZ_BM >> 4) << 24);

struct OzArgs {
  int M, N, kb, ke;        // rows of A / C, rows of B / columns of C, k range [kb, ke)
  int koff;                // global k of this launch's k = 0 (triangular operands, k chunks)
  const int* exA;          // row exponents of A (M) and B (N)
  const int* exB;
  double* C;
  long long ldc;
  double alpha, beta;
  int flags;               // GEMM_A_LOWER / GEMM_B_LOWER / GEMM_C_LOWER
  int gm;                  // row tiles per tile group (oz_tile)
  const int* abort_flag;
  int whatif;              // measurement only (GG_OZ_WHATIF, results invalid): 1 no TMA loads,
                           // 2 no epilogue work
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
      "OZW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra OZW_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
// K-major, 32-byte-swizzled descriptor: rows of 32 B, 8-row groups 256 B apart (SBO), version 1,
// layout SWIZZLE_32B (6)
__device__ __forceinline__ unsigned long long desc32(unsigned saddr) {
  if (OZ_KC == 64)   // rows of 64 B, 8-row groups 512 B apart, layout SWIZZLE_64B (4)
    return (unsigned long long)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (32ull << 32) |
           (1ull << 46) | (4ull << 61);
  return (unsigned long long)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (16ull << 32) |
         (1ull << 46) | (6ull << 61);
}
__device__ __forceinline__ void tma_3d(unsigned dst, const CUtensorMap* map, unsigned bar, int c0,
                                       int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// D[128 x 64 nb] (+)= A . B^T for nb consecutive B slices stacked along N (N = 64 nb <= 256)
__device__ __forceinline__ void mma_i8(unsigned d_tmem, unsigned long long a, unsigned long long b,
                                       int nb, unsigned accumulate) {
  const unsigned idesc = OZ_IDESC_BASE | ((unsigned)(OZ_BN * nb >> 3) << 17);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(unsigned bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ double pow2(int e) {   // 2^e, |e| < 1022
  return __longlong_as_double((long long)(1023 + e) << 52);
}
// 8 columns x the 8 diagonals of one warp quarter: v[d][c]
// the 8 diagonals' accumulators (columns d * OZ_BN) of 8 columns; OZ_S == 7 leaves v[7] unused
__device__ __forceinline__ void tmem_ld_diag8(unsigned taddr, int (&v)[8][8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%64];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%65];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16,%17,%18,%19,%20,%21,%22,%23}, [%66];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%24,%25,%26,%27,%28,%29,%30,%31}, [%67];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%32,%33,%34,%35,%36,%37,%38,%39}, [%68];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%40,%41,%42,%43,%44,%45,%46,%47}, [%69];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%48,%49,%50,%51,%52,%53,%54,%55}, [%70];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%56,%57,%58,%59,%60,%61,%62,%63}, [%71];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(v[0][0]), "=r"(v[0][1]), "=r"(v[0][2]), "=r"(v[0][3]), "=r"(v[0][4]), "=r"(v[0][5]), "=r"(v[0][6]), "=r"(v[0][7]),
        "=r"(v[1][0]), "=r"(v[1][1]), "=r"(v[1][2]), "=r"(v[1][3]), "=r"(v[1][4]), "=r"(v[1][5]), "=r"(v[1][6]), "=r"(v[1][7]),
        "=r"(v[2][0]), "=r"(v[2][1]), "=r"(v[2][2]), "=r"(v[2][3]), "=r"(v[2][4]), "=r"(v[2][5]), "=r"(v[2][6]), "=r"(v[2][7]),
        "=r"(v[3][0]), "=r"(v[3][1]), "=r"(v[3][2]), "=r"(v[3][3]), "=r"(v[3][4]), "=r"(v[3][5]), "=r"(v[3][6]), "=r"(v[3][7]),
        "=r"(v[4][0]), "=r"(v[4][1]), "=r"(v[4][2]), "=r"(v[4][3]), "=r"(v[4][4]), "=r"(v[4][5]), "=r"(v[4][6]), "=r"(v[4][7]),
        "=r"(v[5][0]), "=r"(v[5][1]), "=r"(v[5][2]), "=r"(v[5][3]), "=r"(v[5][4]), "=r"(v[5][5]), "=r"(v[5][6]), "=r"(v[5][7]),
        "=r"(v[6][0]), "=r"(v[6][1]), "=r"(v[6][2]), "=r"(v[6][3]), "=r"(v[6][4]), "=r"(v[6][5]), "=r"(v[6][6]), "=r"(v[6][7]),
        "=r"(v[7][0]), "=r"(v[7][1]), "=r"(v[7][2]), "=r"(v[7][3]), "=r"(v[7][4]), "=r"(v[7][5]), "=r"(v[7][6]), "=r"(v[7][7])
      : "r"(taddr + 0 * OZ_BN), "r"(taddr + 1 * OZ_BN), "r"(taddr + 2 * OZ_BN), "r"(taddr + 3 * OZ_BN),
        "r"(taddr + 4 * OZ_BN), "r"(taddr + 5 * OZ_BN), "r"(taddr + 6 * OZ_BN), "r"(taddr + 7 * OZ_BN)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_diag7(unsigned taddr, int (&v)[8][8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%56];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%57];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16,%17,%18,%19,%20,%21,%22,%23}, [%58];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%24,%25,%26,%27,%28,%29,%30,%31}, [%59];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%32,%33,%34,%35,%36,%37,%38,%39}, [%60];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%40,%41,%42,%43,%44,%45,%46,%47}, [%61];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%48,%49,%50,%51,%52,%53,%54,%55}, [%62];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(v[0][0]), "=r"(v[0][1]), "=r"(v[0][2]), "=r"(v[0][3]), "=r"(v[0][4]), "=r"(v[0][5]), "=r"(v[0][6]), "=r"(v[0][7]),
        "=r"(v[1][0]), "=r"(v[1][1]), "=r"(v[1][2]), "=r"(v[1][3]), "=r"(v[1][4]), "=r"(v[1][5]), "=r"(v[1][6]), "=r"(v[1][7]),
        "=r"(v[2][0]), "=r"(v[2][1]), "=r"(v[2][2]), "=r"(v[2][3]), "=r"(v[2][4]), "=r"(v[2][5]), "=r"(v[2][6]), "=r"(v[2][7]),
        "=r"(v[3][0]), "=r"(v[3][1]), "=r"(v[3][2]), "=r"(v[3][3]), "=r"(v[3][4]), "=r"(v[3][5]), "=r"(v[3][6]), "=r"(v[3][7]),
        "=r"(v[4][0]), "=r"(v[4][1]), "=r"(v[4][2]), "=r"(v[4][3]), "=r"(v[4][4]), "=r"(v[4][5]), "=r"(v[4][6]), "=r"(v[4][7]),
        "=r"(v[5][0]), "=r"(v[5][1]), "=r"(v[5][2]), "=r"(v[5][3]), "=r"(v[5][4]), "=r"(v[5][5]), "=r"(v[5][6]), "=r"(v[5][7]),
        "=r"(v[6][0]), "=r"(v[6][1]), "=r"(v[6][2]), "=r"(v[6][3]), "=r"(v[6][4]), "=r"(v[6][5]), "=r"(v[6][6]), "=r"(v[6][7])
      : "r"(taddr + 0 * OZ_BN), "r"(taddr + 1 * OZ_BN), "r"(taddr + 2 * OZ_BN), "r"(taddr + 3 * OZ_BN),
        "r"(taddr + 4 * OZ_BN), "r"(taddr + 5 * OZ_BN), "r"(taddr + 6 * OZ_BN)
      : "memory");
}

// ---- clusters with multicast operand loads ---------------------------------------------------
// The OZ_CLM x OZ_CLN CTAs of a cluster compute the tiles (mt = OZ_CLM bm + cm, nt = OZ_CLN bn + cn)
// of one block of C in lockstep over the same k range: each A tile is needed by the OZ_CLN CTAs of
// its row (cm) and each B tile by the OZ_CLM CTAs of its column (cn), so every CTA loads its share
// of the slices (4 per load) and multicasts them to the CTAs that need them.  A stage is freed
// for the producer of CTA X only when X and every CTA it multicasts into have consumed it: each
// CTA's MMA commit arrives on the "empty" barriers of the CTAs sharing its A or B tile.
// Measured (r02, tools/prof_ozaki.py, same box, round-robin): 1 x 2 (the A tile shared by two
// column-neighbour CTAs: a third less L2->SM traffic, 74 resident clusters) 5-14% faster than
// independent CTAs; 2 x 2 fits only 33 resident clusters of 4 (GPC packing: 132 SMs) and 2 x 1
// shares the smaller B tile -- both slower.  What-if (GG_OZ_WHATIF=1, no operand loads): +34-46%
// on the long-k GEMMs, so the loads remain the limiter.
#ifndef OZ_CLM
#define OZ_CLM 1
#endif
#ifndef OZ_CLN
#define OZ_CLN 2
#endif
constexpr int OZ_CL = OZ_CLM * OZ_CLN;                        // CTAs per cluster
constexpr int OZ_CBM = OZ_CLM * OZ_BM, OZ_CBN = OZ_CLN * OZ_BN;   // cluster block of C

// blocks in groups of a.gm block rows swept block column by block column (the concurrently running
// blocks share ~gm A row panels: L2 reuse); triangular A: heavy (last) block rows first.  A
// group's column range: all num_bn, or for a lower C up to the diagonal of its last block row.
__device__ __forceinline__ int oz_group_nb(const OzArgs& a, int g, int num_bm, int num_bn) {
  if (!(a.flags & GEMM_C_LOWER)) return num_bn;
  const int lo = g * a.gm, hi = min(num_bm, lo + a.gm) - 1;
  const int bm_max = (a.flags & GEMM_A_LOWER) ? num_bm - 1 - lo : hi;
  return min(num_bn, (OZ_CBM * bm_max + OZ_CBM + OZ_CBN - 1) / OZ_CBN);   // n0 < m0 + CBM
}
__device__ __forceinline__ int oz_total(const OzArgs& a, int num_bm, int num_bn) {
  int tot = 0;
  for (int g = 0; g * a.gm < num_bm; ++g)
    tot += min(a.gm, num_bm - g * a.gm) * oz_group_nb(a, g, num_bm, num_bn);
  return tot;
}
// block t -> (bm, bn) and the block's k range (the union of its tiles' ranges: operand entries
// outside a tile's own triangle are zero slices); false when the block lies above the diagonal
__device__ __forceinline__ bool oz_block(const OzArgs& a, int t, int num_bm, int num_bn, int& bm,
                                         int& bn, int& kb, int& ke) {
  int g = 0, gm = 0, gn = 0;
  for (;; ++g) {
    gm = min(a.gm, num_bm - g * a.gm);
    gn = oz_group_nb(a, g, num_bm, num_bn);
    if (t < gm * gn) break;
    t -= gm * gn;
  }
  bn = t / gm;
  const int lin = g * a.gm + t % gm;
  bm = (a.flags & GEMM_A_LOWER) ? num_bm - 1 - lin : lin;
  const int m0 = bm * OZ_CBM, n0 = bn * OZ_CBN;
  if ((a.flags & GEMM_C_LOWER) && n0 >= m0 + OZ_CBM) return false;
  kb = a.kb;
  ke = a.ke;
  if (a.flags & GEMM_A_LOWER) ke = min(ke, m0 + OZ_CBM - a.koff);   // A(i, k) = 0 for k > i
  if (a.flags & GEMM_B_LOWER) kb = max(kb, n0 - a.koff);            // B(j, k) = 0 for k < j
  return true;
}

__device__ __forceinline__ unsigned cta_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" :::
                   "memory");
}
__device__ __forceinline__ void tma_3d_mc(unsigned dst, const CUtensorMap* map, unsigned bar, int c0,
                                          int c1, int c2, unsigned short mask) {
  if (OZ_CL == 1) {
    tma_3d(dst, map, bar, c0, c1, c2);
    return;
  }
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4, %5}], [%2], %6;\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(unsigned bar, unsigned short mask) {
  if (OZ_CL == 1) {
    mma_commit(bar);
    return;
  }
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;\n" ::"r"(bar),
      "h"(mask)
      : "memory");
}

__global__ void __launch_bounds__(OZ_THREADS, 1)
    ozaki_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      OzArgs a) {
  if (a.abort_flag != nullptr && *a.abort_flag != 0) return;   // uniform across the grid
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(smem + OZ_STAGES * OZ_STAGE_BYTES);
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(bars + 2 * OZ_STAGES + 2);
  const unsigned sbase = smem_u32(smem);
  const unsigned full0 = smem_u32(bars), empty0 = full0 + 8 * OZ_STAGES;
  const unsigned accf = empty0 + 8 * OZ_STAGES, acce = accf + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned rank = OZ_CL > 1 ? cta_rank() : 0u;
  const int cm = rank % OZ_CLM, cn = rank / OZ_CLM;
  unsigned short mask_a = 0, mask_b = 0;   // the CTAs sharing this CTA's A tile (same cm) / B tile
  for (int i = 0; i < OZ_CLN; ++i) mask_a |= (unsigned short)(1u << (cm + OZ_CLM * i));
  for (int i = 0; i < OZ_CLM; ++i) mask_b |= (unsigned short)(1u << (i + OZ_CLM * cn));
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, OZ_CLM + OZ_CLN - 1);
    }
    mbar_init(accf, 1);
    mbar_init(acce, OZ_EPI_WARPS * 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  fence_before();
  if (OZ_CL > 1) cluster_sync_all();   // barriers initialised in every CTA before any multicast
  else __syncthreads();
  fence_after();
  const unsigned tmem_base = *tmem_slot;
  const int num_mt = (a.M + OZ_BM - 1) / OZ_BM, num_nt = (a.N + OZ_BN - 1) / OZ_BN;
  const int num_bm = (num_mt + OZ_CLM - 1) / OZ_CLM, num_bn = (num_nt + OZ_CLN - 1) / OZ_CLN;
  const int total = oz_total(a, num_bm, num_bn);
  const int cid = blockIdx.x / OZ_CL, ncl = gridDim.x / OZ_CL;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      for (int t = cid; t < total; t += ncl) {
        int bm, bn, kb, ke;
        if (!oz_block(a, t, num_bm, num_bn, bm, bn, kb, ke)) continue;
        for (int k = kb; k < ke; k += OZ_KC) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const unsigned fb = full0 + 8 * stage, dA = sbase + stage * OZ_STAGE_BYTES;
          if (a.whatif & 1) {
            mbar_arrive(fb);
          } else {
            mbar_expect_tx(fb, OZ_STAGE_BYTES);
            // this CTA's share of its A tile's slices (4 per load) and of its B tile's
            for (int q = cn * (2 / OZ_CLN); q < (cn + 1) * (2 / OZ_CLN); ++q)
              tma_3d_mc(dA + 4 * q * (OZ_BM * OZ_KC), &tmA, fb, k, (OZ_CLM * bm + cm) * OZ_BM,
                        4 * q, mask_a);
            for (int q = cm * (2 / OZ_CLM); q < (cm + 1) * (2 / OZ_CLM); ++q)
              tma_3d_mc(dA + OZ_A_BYTES + 4 * q * (OZ_BN * OZ_KC), &tmB, fb, k,
                        (OZ_CLN * bn + cn) * OZ_BN, 4 * q, mask_b);
          }
          if (++stage == OZ_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      int it = 0;
      for (int t = cid; t < total; t += ncl) {
        int bm, bn, kb, ke;
        if (!oz_block(a, t, num_bm, num_bn, bm, bn, kb, ke)) continue;
        if (ke <= kb) continue;
        mbar_wait(acce, (it & 1) ^ 1);   // the epilogue has the previous tile in registers
        fence_after();
        for (int k = kb; k < ke; k += OZ_KC) {
          mbar_wait(full0 + 8 * stage, phase);
          fence_after();
          const unsigned sA = sbase + stage * OZ_STAGE_BYTES, sB = sA + OZ_A_BYTES;
          // A slice s times B slices u = 0 .. OZ_S-1-s: the B slices sit consecutively along N,
          // and product (s, u) belongs to diagonal s + u at TMEM column 64 (s + u), so one MMA
          // covers up to 4 of them (N = 256): 10 MMAs per K step for the 28 products (12 for 36
          // with 7-bit digits), so the tensor core reads each A slice from shared memory once or
          // twice rather than OZ_S - s times.  s = 0 opens every diagonal.
#pragma unroll
          for (int kk = 0; kk < OZ_KC / 32; ++kk) {   // MMA K steps of 32 bytes in the stage
#pragma unroll
            for (int s = 0; s < OZ_S; ++s) {
              const unsigned long long da = desc32(sA + s * (OZ_BM * OZ_KC)) + 2 * kk;
              // 8 - s products in one or two MMAs, split evenly (N = 64 runs at 62% of the int8
              // rate on this B200 -- shared-memory bound -- N = 128..256 at 94-100%, tools/i8_peak)
              const int cnt = OZ_S - s;
              const int first = cnt > 4 ? (cnt + 1) / 2 : cnt;
              const unsigned acc = (k > kb || kk > 0 || s > 0) ? 1u : 0u;
              mma_i8(tmem_base + s * OZ_BN, da, desc32(sB) + 2 * kk, first, acc);
              if (cnt > first)
                mma_i8(tmem_base + (s + first) * OZ_BN, da,
                       desc32(sB + first * (OZ_BN * OZ_KC)) + 2 * kk, cnt - first, acc);
            }
          }
          mma_commit_mc(empty0 + 8 * stage, mask_a | mask_b);
          if (++stage == OZ_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(accf);
        ++it;
      }
    }
  } else {
    // 8 epilogue warps: warp w reads TMEM lanes 32 (w % 4) .. +31 (its tile rows) and half h of
    // the tile's 64 columns, so the accumulators are released twice as fast as with 4 warps
    const int quarter = warp & 3, h = (warp - 2) >> 2;
    const int row_l = quarter * 32 + lane;
    int it = 0;
    for (int t = cid; t < total; t += ncl) {
      int bm, bn, kb, ke;
      if (!oz_block(a, t, num_bm, num_bn, bm, bn, kb, ke)) continue;
      const int mt = OZ_CLM * bm + cm, nt = OZ_CLN * bn + cn;
      const bool write = mt < num_mt && nt < num_nt &&
                         !((a.flags & GEMM_C_LOWER) && nt * OZ_BN >= mt * OZ_BM + OZ_BM);
      const int row = mt * OZ_BM + row_l, n0 = nt * OZ_BN + h * (OZ_BN / 2);
      constexpr int HN = OZ_BN / 2;
      double r[HN];
      if (ke > kb) {
        mbar_wait(accf, it & 1);
        fence_after();
        if (!(a.whatif & 2)) {
          const unsigned taddr = tmem_base + ((unsigned)(quarter * 32) << 16) + h * HN;
#pragma unroll
          for (int c8 = 0; c8 < HN / 8; ++c8) {
            int v[8][8];
            if (OZ_S == 8) tmem_ld_diag8(taddr + c8 * 8, v);
            else tmem_ld_diag7(taddr + c8 * 8, v);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              if (OZ_DB == 7) {   // sum_d D_d 2^(-7 (d+2)): exact halves in base 2^7
                const long long hi = (((long long)v[0][c] * 128 + v[1][c]) * 128 + v[2][c]) * 128 +
                                     v[3][c];
                const long long lo = (((long long)v[4][c] * 128 + v[5][c]) * 128 + v[6][c]) * 128 +
                                     v[7][c];
                r[c8 * 8 + c] = fma((double)hi, 0x1p-35, (double)lo * 0x1p-63);   // the one rounding
              } else {            // sum_d D_d 2^(-8 (d+2)): |hi| < 2^52, |lo| < 2^46, both exact
                const long long hi = (((long long)v[0][c] * 256 + v[1][c]) * 256 + v[2][c]) * 256 +
                                     v[3][c];
                const long long lo = ((long long)v[4][c] * 256 + v[5][c]) * 256 + v[6][c];
                r[c8 * 8 + c] = fma((double)hi, 0x1p-40, (double)lo * 0x1p-64);   // the one rounding
              }
            }
          }
        }
        fence_before();
        mbar_arrive(acce);
        ++it;
        if (a.whatif & 2) continue;
        // scale by 2^(e_i + f_j) after the accumulators are released: exact for normal results
        // (the same bits as rounding at the final scale); ldexp gives the IEEE inf / subnormal
        // at the ends of the exponent range
        const int ea = row < a.M ? max(a.exA[row], -4000) : 0;   // EX_NONE: all-zero row
#pragma unroll
        for (int c = 0; c < HN; ++c) {
          const int col = n0 + c;
          const int e = ea + (col < a.N ? max(__ldg(a.exB + col), -4000) : 0);
          r[c] = (e > -1000 && e < 1000) ? r[c] * pow2(e) : ldexp(r[c], e);
        }
      } else {
#pragma unroll
        for (int c = 0; c < HN; ++c) r[c] = 0.0;
      }
      if (write && row < a.M) {   // C = beta C + alpha r in chunks of 8 columns, next chunk's loads in flight
        constexpr int CH = 8;
        double* cbase = a.C + (long long)n0 * a.ldc + row;
        const int ncol = min(HN, a.N - n0);
        const bool rd = a.beta != 0.0;
        double cv[CH], cn_[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) cv[c] = (rd && c < ncol) ? cbase[(long long)c * a.ldc] : 0.0;
#pragma unroll
        for (int ch = 0; ch < HN / CH; ++ch) {
          if (ch + 1 < HN / CH) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              const int cc = (ch + 1) * CH + c;
              cn_[c] = (rd && cc < ncol) ? cbase[(long long)cc * a.ldc] : 0.0;
            }
          }
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const int cc = ch * CH + c;
            if (cc < ncol)
              cbase[(long long)cc * a.ldc] = rd ? fma(a.alpha, r[cc], a.beta * cv[c]) : a.alpha * r[cc];
          }
#pragma unroll
          for (int c = 0; c < CH; ++c) cv[c] = cn_[c];
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (OZ_CL > 1) cluster_sync_all();   // no peer multicast / remote arrive may target an exited CTA
  fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem_base)
                 : "memory");
  }
}

// ---- slicing -----------------------------------------------------------------------------------
// X(r, k) = X[r rs + k cs], rows [0, R), k in [0, K).  Tiles of TR rows x TK k (4,096 elements)
// staged through shared memory with the coalesced thread mapping for whichever stride is 1:
// 128 x 32 when the rows are contiguous (1 KB runs per column -- 32-row tiles read 256-B runs
// 320 KB apart and streamed at ~1.7 TB/s on the 39k-row SYRK operand at n = 4e4), 32 x 128 when
// k is.
constexpr int SL_THREADS = 256;
constexpr int EX_NONE = (int)0x80808080;  // row-exponent sentinel (memset 0x80): no nonzero yet
__device__ __forceinline__ int tix(int k) { return k + (k >> 4); }   // one pad per 16 k

template <int TR, int TK>
__device__ __forceinline__ void load_tile(double (*T)[TK + TK / 16], const double* __restrict__ X,
                                          long long rs, long long cs, int R, int K, int r0,
                                          int k0) {
  // all of a thread's 16 loads are issued before the first shared-memory store (r02 end: one
  // load in flight per thread left these kernels HBM-latency-bound at ~2.5 TB/s)
  constexpr int PER = TR * TK / SL_THREADS;
  static_assert(PER * SL_THREADS == TR * TK, "whole tile per pass");
  double v[PER];
  if (rs <= cs) {   // rows contiguous: consecutive threads -> consecutive rows
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * SL_THREADS;
      const int r = i % TR, k = i / TR;
      v[j] = (r0 + r < R && k0 + k < K)
                 ? X[(long long)(r0 + r) * rs + (long long)(k0 + k) * cs] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * SL_THREADS;
      T[i % TR][tix(i / TR)] = v[j];
    }
  } else {          // k contiguous: consecutive threads -> consecutive k
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * SL_THREADS;
      const int k = i % TK, r = i / TK;
      v[j] = (r0 + r < R && k0 + k < K)
                 ? X[(long long)(r0 + r) * rs + (long long)(k0 + k) * cs] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * SL_THREADS;
      T[i / TK][tix(i % TK)] = v[j];
    }
  }
}

// triangular operands (flags of ozaki_gemm_run): entries outside the triangle are taken as zero
// whatever the memory holds -- tri 1: A~(i, k) = 0 for k > i; tri 2: B~(j, k) = 0 for k < j
// (k global: the chunk offset added)
__device__ __forceinline__ bool oz_masked(int tri, int r, int k) {
  return (tri == 1 && k > r) || (tri == 2 && k < r);
}

// ex[r] = max(ex[r], e) with max_k |X(r,k)| < 2^e over this CTA's tile (ex starts at EX_NONE; the
// exponent of the row maximum is the maximum of the tile exponents); each warp reduces TR / 8
// rows of the staged tile (r02: a thread per row walking 256 strided k values was latency-bound).
template <int TR, int TK>
__global__ void __launch_bounds__(SL_THREADS) oz_rowexp_kernel(int R, int K, const double* X,
                                                                long long rs, long long cs,
                                                                int* ex, int tri, int koff,
                                                                const int* abort_flag) {
  if (abort_flag != nullptr && *abort_flag != 0) return;
  __shared__ double T[TR][TK + TK / 16];
  const int r0 = blockIdx.x * TR, k0 = blockIdx.y * TK;
  load_tile<TR, TK>(T, X, rs, cs, R, K, r0, k0);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int rr = warp; rr < TR; rr += SL_THREADS / 32) {
    const int r = r0 + rr;
    if (r >= R) break;
    double m = 0.0;
#pragma unroll
    for (int j = 0; j < TK / 32; ++j) {
      const int k = lane + 32 * j;
      if (!oz_masked(tri, r, koff + k0 + k)) m = fmax(m, fabs(T[rr][tix(k)]));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0 && m > 0.0) {
      int e;
      const double mant = frexp(m, &e);   // m = mant 2^e, mant in [0.5, 1)
      // 8-bit balanced digits need |x| 2^-e < 127/256 (the top digit stays <= 127): monotone in
      // m, so the maximum over tiles is the exponent of the row maximum
      if (OZ_DB == 8) e += mant < 127.0 / 128.0 ? 1 : 2;
      atomicMax(ex + r, e);
    }
  }
}

// Sl[s][r][k] (row stride kp bytes, slice stride kp * R) for k in [0, kp): exact slices below 2^ex[r];
// 16 consecutive k per thread (TK / 16 threads per row)
template <int TR, int TK>
__global__ void __launch_bounds__(SL_THREADS) oz_slice_kernel(int R, int K, const double* X,
                                                               long long rs, long long cs,
                                                               const int* ex, signed char* Sl,
                                                               long long kp, int tri, int koff,
                                                               const int* abort_flag) {
  static_assert(TR * (TK / 16) == SL_THREADS, "one 16-k run per thread");
  if (abort_flag != nullptr && *abort_flag != 0) return;
  __shared__ double T[TR][TK + TK / 16];
  const int r0 = blockIdx.x * TR, k0 = blockIdx.y * TK;
  load_tile<TR, TK>(T, X, rs, cs, R, K, r0, k0);
  __syncthreads();
  const int r = threadIdx.x / (TK / 16), kq = (threadIdx.x % (TK / 16)) * 16;
  if (r0 + r >= R || k0 + kq >= kp) return;
  const int ee = ex[r0 + r];
  const int e = ee == EX_NONE ? 0 : ee;   // all-zero row
  unsigned w[OZ_S][4] = {};
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double x = T[r][tix(kq + j)];
    // |v| < 1; 2^-e by its bits (exact) unless the row sits at the ends of the exponent range
    const double v = oz_masked(tri, r0 + r, koff + k0 + kq + j) ? 0.0
                     : (e > -1000 && e < 1000) ? x * pow2(-e) : ldexp(x, -e);
    // digits of the magnitude |v| 2^56 (rounded to nearest once: the last slice's rounding) in
    // base 128, each carrying the element's sign -- the truncated digits of v: the dropped
    // products (s + t >= 8) and the residuals keep random signs and cancel along k (floor digits
    // -- all non-negative below slice 0 -- make them add up coherently: measured 30-90x larger
    // GEMM errors).  One FP64 -> integer conversion per element, the rest integer work.
    if (OZ_DB == 7) {
      const unsigned long long N = __double2ull_rn(fabs(v) * 0x1p56);   // exact scale, < 2^56
      const bool neg = v < 0.0;
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) {
        const int d = (int)((N >> (7 * (OZ_S - 1 - s))) & 127u);
        w[s][j / 4] |= ((unsigned)(neg ? -d : d) & 0xffu) << (8 * (j % 4));
      }
    } else {
      // balanced base-256 digits of V = RN(v 2^56) (|v| < 127/256: the top digit in [-127, 127]),
      // lowest first; every digit below the top one is centred on zero, so the dropped products
      // (s + t >= 7) keep random signs and cancel along k like the sign-magnitude digits
      long long V = __double2ll_rn(v * 0x1p56);
#pragma unroll
      for (int s = OZ_S - 1; s > 0; --s) {
        const int d = (int)((V + 128) & 255) - 128;
        V = (V - d) >> 8;
        w[s][j / 4] |= ((unsigned)d & 0xffu) << (8 * (j % 4));
      }
      w[0][j / 4] |= ((unsigned)(int)V & 0xffu) << (8 * (j % 4));
    }
  }
  const long long off = (long long)(r0 + r) * kp + k0 + kq;
#pragma unroll
  for (int s = 0; s < OZ_S; ++s)
    *reinterpret_cast<uint4*>(Sl + (long long)s * kp * R + off) =
        make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_oz() {
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

int encode_slices(CUtensorMap* map, const signed char* Sl, int R, int K, long long kp, int box_rows) {
  auto fn = encode_fn_oz();
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  if (const char* v = getenv("GG_OZ_PROMO"))   // tuning knob: 0 none, 1 64B, 2 128B, 3 256B
    promo = (CUtensorMapL2promotion)atoi(v);
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return GG_ECUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)R, (cuuint64_t)OZ_S};
  cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)kp * R};
  cuuint32_t box[3] = {OZ_KC, (cuuint32_t)box_rows, OZ_SS / 2};   // half the slots (multicast)
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<signed char*>(Sl), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  OZ_KC == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                  promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (ozaki slices) failed (code " + std::to_string((int)r) + ")");
    return GG_ECUDA;
  }
  return GG_OK;
}

inline long long oz_kp(int K) { return ((long long)(K < OZ_KMAX ? K : OZ_KMAX) + 15) / 16 * 16; }
inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
inline size_t oz_operand_bytes(int R, int K) {
  return align256((size_t)OZ_S * R * oz_kp(K)) + align256((size_t)R * sizeof(int));
}

// clusters of 4 that can be resident at once (GPCs hold whole clusters: fewer than 148 / 4)
int oz_max_clusters() {
  static std::once_flag once;
  static int n = 0;
  std::call_once(once, [] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(OZ_CL * (148 / OZ_CL));
    cfg.blockDim = dim3(OZ_THREADS);
    cfg.dynamicSmemBytes = OZ_SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = OZ_CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaFuncSetAttribute(ozaki_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)OZ_SMEM) != cudaSuccess ||
        cudaOccupancyMaxActiveClusters(&n, ozaki_gemm_kernel, &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 1;
    }
    if (getenv("GG_OZ_VERBOSE")) fprintf(stderr, "[gg ozaki] %d resident clusters of %d\n", n, OZ_CL);
  });
  return n;
}


int slice_operand(int R, int Kc, const double* X, long long rs, long long cs, signed char* Sl,
                  int* ex, long long kp, int tri, int koff, const int* abort_flag, cudaStream_t s) {
  GG_CUDA_TRY(cudaMemsetAsync(ex, 0x80, (size_t)R * sizeof(int), s));   // EX_NONE
  auto run = [&](auto tr, auto tk) {
    constexpr int TR = decltype(tr)::value, TK = decltype(tk)::value;
    const dim3 gx((R + TR - 1) / TR, (Kc + TK - 1) / TK);
    oz_rowexp_kernel<TR, TK><<<gx, SL_THREADS, 0, s>>>(R, Kc, X, rs, cs, ex, tri, koff, abort_flag);
    const dim3 g((R + TR - 1) / TR, (unsigned)((kp + TK - 1) / TK));
    oz_slice_kernel<TR, TK><<<g, SL_THREADS, 0, s>>>(R, Kc, X, rs, cs, ex, Sl, kp, tri, koff,
                                                     abort_flag);
  };
  if (rs <= cs)
    run(std::integral_constant<int, 128>(), std::integral_constant<int, 32>());
  else
    run(std::integral_constant<int, 32>(), std::integral_constant<int, 128>());
  GG_LAUNCH_CHECK("oz_slice_kernel");
  return GG_OK;
}

}  // namespace

size_t ozaki_ws_bytes(int M, int N, int K, bool b_is_a) {
  return oz_operand_bytes(M, K) + (b_is_a ? 0 : oz_operand_bytes(N, K));
}

int ozaki_gemm_run(int M, int N, int K, const double* A, long long a_rs, long long a_cs,
                   const double* B, long long b_rs, long long b_cs, double* C, long long ldc,
                   double alpha, double beta, int flags, void* ws, size_t ws_bytes,
                   const int* abort_flag, cudaStream_t s) {
  if (M <= 0 || N <= 0) return GG_OK;
  const bool same = (B == nullptr);
  if (same && N > M) {   // B~ = the first N rows of A~ (N < M: a SYRK on leading columns)
    set_error("ozaki_gemm: B = A needs N <= M");
    return GG_EDIM;
  }
  if (ws == nullptr || ws_bytes < ozaki_ws_bytes(M, N, K, same)) {
    set_error("ozaki_gemm: workspace too small");
    return GG_EARG;
  }
  if (K <= 0) {   // C = beta C: the GEMM with an empty k range
    if (beta == 1.0) return GG_OK;
    set_error("ozaki_gemm: K == 0 with beta != 1 is not supported");
    return GG_EARG;
  }
  const long long kp = oz_kp(K);
  signed char* SlA = static_cast<signed char*>(ws);
  int* exA = reinterpret_cast<int*>(static_cast<char*>(ws) + align256((size_t)OZ_S * M * kp));
  signed char* SlB = SlA;
  int* exB = exA;
  if (!same) {
    SlB = static_cast<signed char*>(ws) + oz_operand_bytes(M, K);
    exB = reinterpret_cast<int*>(reinterpret_cast<char*>(SlB) + align256((size_t)OZ_S * N * kp));
  }
  GG_CUDA_TRY(cudaFuncSetAttribute(ozaki_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)OZ_SMEM));
  // k chunks of at most OZ_KMAX (exact int32 diagonals); beta applies to the first chunk only
  for (int k0 = 0; k0 < K; k0 += OZ_KMAX) {
    const int Kc = (K - k0 < OZ_KMAX) ? (K - k0) : OZ_KMAX;
    // (B = A: the SYRK, no triangle flags on its operand)
    int rc = slice_operand(M, Kc, A + (long long)k0 * a_cs, a_rs, a_cs, SlA, exA, kp,
                           (flags & GEMM_A_LOWER) ? 1 : 0, k0, abort_flag, s);
    if (rc != GG_OK) return rc;
    if (!same) {
      rc = slice_operand(N, Kc, B + (long long)k0 * b_cs, b_rs, b_cs, SlB, exB, kp,
                         (flags & GEMM_B_LOWER) ? 2 : 0, k0, abort_flag, s);
      if (rc != GG_OK) return rc;
    }
    CUtensorMap mA, mB;
    rc = encode_slices(&mA, SlA, M, Kc, kp, OZ_BM);
    if (rc != GG_OK) return rc;
    rc = encode_slices(&mB, SlB, same ? M : N, Kc, kp, OZ_BN);
    if (rc != GG_OK) return rc;
    OzArgs a{};
    a.M = M;
    a.N = N;
    // triangular operands: k is relative to this chunk; the row/column offsets of the triangle
    // move with the chunk start
    a.kb = 0;
    a.ke = Kc;
    a.koff = k0;
    a.exA = exA;
    a.exB = exB;
    a.C = C;
    a.ldc = ldc;
    a.alpha = alpha;
    a.beta = (k0 == 0) ? beta : 1.0;
    a.flags = flags;
    a.gm = 8;
    if (const char* v = getenv("GG_OZ_GM")) a.gm = atoi(v) > 0 ? atoi(v) : 8;   // tuning knob
    a.abort_flag = abort_flag;
    if (const char* v = getenv("GG_OZ_WHATIF")) a.whatif = atoi(v);
    const long long blocks = (long long)((M + OZ_CBM - 1) / OZ_CBM) * ((N + OZ_CBN - 1) / OZ_CBN);
    const int resident = oz_max_clusters();   // a persistent grid must be co-resident
    const int clusters = (int)(blocks < resident ? blocks : resident);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(OZ_CL * clusters);
    cfg.blockDim = dim3(OZ_THREADS);
    cfg.dynamicSmemBytes = OZ_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = OZ_CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GG_CUDA_TRY(cudaLaunchKernelEx(&cfg, ozaki_gemm_kernel, mA, mB, a));
  }
  return GG_OK;
}

}  // namespace gg
